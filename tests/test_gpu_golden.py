"""Full-size parity of the B200 path against the oracle's golden fixtures.

tests/golden/cfg<c>.npz were produced by tools/make_golden.py, which runs the
CPU oracle (the restatement of the reference hot path) on BASELINE config c at
its full size and seed (cfg3 / cfg4 on the GPU box's host: see
tests/golden/README.md).  Here the GPU path builds the same config through
the C ABI and is compared at north_star's tolerances:

  element ItI maps and sources  <= 1e-10 (relative Frobenius; every element
                                 through seeded sketches, sampled elements in full)
  every level system M_l         <= 1e-10 (relative, y = M_l r sketched)
  MG(v), rhs                     <= 1e-10
  FGMRES solution                <= 1e-9 (relative L2, sketched)
  FGMRES iteration count         +-1

A sketch of a vector y is W^H y with W a seeded dim x 8 complex Gaussian
matrix; of a map T it is w^H T r with seeded unit-variance w, r, whose RMS
over w, r is ||T||_F -- so relative sketch differences estimate the relative
errors above (tools/make_golden.py).
"""
import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import make_golden as mg  # noqa: E402  (seeded sketch vectors, shared with the generator)

pytestmark = pytest.mark.gpu

TOL_OP = 1e-10
TOL_SOL = 1e-9
GOLDEN = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "cfg*.npz")))
CONFIGS = [int(os.path.basename(p)[3:-4]) for p in GOLDEN]


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


class Run:
    """The GPU pipeline of one config at full size (built once per config)."""

    def __init__(self, hps, c):
        self.g = np.load(os.path.join(ROOT, "tests", "golden", f"cfg{c}.npz"))
        self.meta = json.loads(str(self.g["meta"]))
        self.prob = hps.problem(2, c, seed=self.meta["seed"])
        assert (self.prob.n, self.prob.order) == (self.meta["n"], self.meta["order"])
        self.ctx = hps.Context(0)
        self.el = hps.build_elements(self.ctx, self.prob)
        self.sk = hps.assemble_skeleton(self.el, self.prob)
        assert self.sk.dim == self.meta["dim"]
        self.hier = hps.build_hierarchy(self.sk, factor_coarse=False)
        m = self.meta["mg"]
        self.pc = hps.build_preconditioner(self.hier, depth=m["depth"], gamma=m["gamma"],
                                           coarse_iters=m["coarse_iters"])

    def close(self):
        for name in ("pc", "hier", "sk", "el"):
            getattr(self, name).close()
        self.ctx.close()


@pytest.fixture(scope="module", params=CONFIGS, ids=[f"cfg{c}" for c in CONFIGS])
def run(request):
    import paper_2511_00735_b200 as hps
    r = Run(hps, request.param)
    yield r
    r.close()


def test_elements(run):
    g, nb = run.g, run.el.nb
    ne = run.prob.n ** 2
    wT, rT, wH = mg.elem_vectors(nb)
    worst_t = worst_h = 0.0
    chunk = 4096
    for e0 in range(0, ne, chunk):
        T, H = run.el.iti(e0, min(chunk, ne - e0))
        for p in range(2):
            s = np.einsum("i,eij,j->e", wT[p].conj(), T, rT[p])
            worst_t = max(worst_t, np.max(np.abs(s - g["sT"][e0:e0 + len(T), p]) /
                                          g["nT"][e0:e0 + len(T)]))
        sh = H @ wH.conj()
        nh = g["nH"][e0:e0 + len(T)]
        if np.any(nh > 0):
            worst_h = max(worst_h, np.max(np.abs(sh - g["sH"][e0:e0 + len(T)])[nh > 0] / nh[nh > 0]))
        else:
            assert np.all(H == 0)  # s = 0 gives exactly zero H (cfg4)
    assert worst_t < TOL_OP, worst_t
    assert worst_h < TOL_OP, worst_h
    for k, e in enumerate(g["elem_ids"]):
        T, H = run.el.iti(int(e), 1)
        assert rel(T[0], g["T_samples"][k]) < TOL_OP, e
        if np.linalg.norm(g["H_samples"][k]) > 0:
            assert rel(H[0], g["H_samples"][k]) < TOL_OP, e


def test_rhs(run):
    for b, q in enumerate(run.g["q_rhs_b"]):
        assert rel(mg.sketch(201, run.sk.rhs(b)), q) < TOL_OP, b


def test_level_systems(run):
    g = run.g
    assert run.hier.depth == run.meta["levels"] == len(g["q_levels"])
    import paper_2511_00735_b200 as hps
    lr = hps.face_graph(run.prob.n)["level_range"]
    nf = 2 * run.prob.n * (run.prob.n - 1)
    for level in range(1, run.hier.depth + 1):
        dim_l = (nf - int(lr[level - 1][0])) * 2 * run.el.m
        y = run.hier.level_apply(level, mg.level_input(level, dim_l))
        assert abs(np.linalg.norm(y) / g["n_levels"][level - 1] - 1) < 1e-9, level
        assert rel(mg.sketch(2000 + level, y), g["q_levels"][level - 1]) < TOL_OP, level


def test_preconditioner_apply(run):
    z = run.pc.apply(mg.mg_input(run.sk.dim))
    assert rel(mg.sketch(3001, z), run.g["q_mg"]) < TOL_OP


def test_fgmres(run):
    """FGMRES with the reference driver's settings (driver.cpp:125-132):
    iterations within +-1 and the solution within 1e-9 for every right-hand
    side in the fixture (cfg4: its first 4, solved together as a multi-RHS
    batch)."""
    import paper_2511_00735_b200 as hps
    g, meta = run.g, run.meta
    R = meta["rhs"]
    if R == 1:
        x, rep = hps.fgmres(run.sk, run.sk.rhs(0), run.pc, restart=meta["restart"],
                            tol=meta["tol"], record_history=True)
        reps, X = [rep], [x]
        hist = np.asarray(rep["residual_history"])
        ho = g["history_0"]
        k = min(len(hist), len(ho))
        # the residual estimates follow the oracle's curve (to rounding growth)
        assert np.all(np.abs(np.log10(hist[:k] / ho[:k])) < 0.1), (hist[:k], ho[:k])
    else:
        rhs = np.stack([run.sk.rhs(b) for b in range(R)])
        X, reps = hps.fgmres_batch(run.sk, rhs, run.pc, restart=meta["restart"], tol=meta["tol"])
    for b in range(R):
        assert reps[b]["converged"], (b, reps[b])
        assert abs(reps[b]["iterations"] - int(g["iterations"][b])) <= 1, \
            (b, reps[b]["iterations"], int(g["iterations"][b]))
        assert rel(mg.sketch(4001, X[b]), g["q_x"][b]) < TOL_SOL, b
        assert abs(np.linalg.norm(X[b]) / g["n_x"][b] - 1) < TOL_SOL, b
