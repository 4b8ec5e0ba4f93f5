#!/usr/bin/env python3
"""Golden fixtures for the full-size parity tests (tests/golden/cfg<c>.npz).

TEST INFRASTRUCTURE: runs the CPU oracle (oracle/, the restatement of the
reference hps2d hot path) on a BASELINE config at its FULL size and seed and
records what the GPU path must reproduce, in a form small enough to commit:

  * every element's ItI map T_e and source H_e through seeded random sketches
    s_e = w^H T_e r (2 pairs) and w^H H_e, plus ||T_e||_F, ||H_e||; the full
    maps of a few sampled elements;
  * every level system M_l (HierarchyLevel::M, dissection.cpp:200-227) through
    y = M_l r_l for a seeded r_l, sketched as W_l^H y (8 columns) and ||y||;
  * the right-hand side, MG(v) for a seeded v (MgPreconditioner::apply with
    depth = L, gamma = 1, coarse_iters = 4: the reference driver defaults,
    driver.hpp:30-32) and the FGMRES solution (reorthogonalize on,
    driver.cpp:125-132), each sketched the same way;
  * the FGMRES iteration count, final residual and residual history.

For a complex Gaussian w, r with unit-variance entries, E|w^H E r|^2 =
||E||_F^2, so a sketch difference measures the Frobenius / 2-norm error of
the sketched object; tests/test_gpu_golden.py regenerates the same seeded
vectors (numpy PCG64, portable) and compares at north_star's tolerances.

  python tools/make_golden.py --config 2 [--rhs 1] [--threads 16] [--out tests/golden]

cfg3 needs ~90 GB of host memory (the oracle stores M_l in the reference's
block layout), so it is generated on the GPU box's host; see
tests/golden/README.md for the commands and run times.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KAPPA = [10.0, 40.0, 160.0, 400.0, 600.0]
RESTART = [50, 50, 100, 100, 60]
TOL = [1e-10, 1e-10, 1e-10, 1e-10, 1e-8]
NSK = 8  # sketch columns for vectors


def cgauss(rng, shape):
    """Complex Gaussian with unit-variance entries."""
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2.0)


def elem_vectors(nb: int):
    rng = np.random.default_rng(101)
    return cgauss(rng, (2, nb)), cgauss(rng, (2, nb)), cgauss(rng, nb)


def sketch_matrix(seed: int, dim: int) -> np.ndarray:
    return cgauss(np.random.default_rng(seed), (dim, NSK))


def sketch(seed: int, y: np.ndarray) -> np.ndarray:
    return sketch_matrix(seed, y.shape[0]).conj().T @ y


def level_input(level: int, dim: int) -> np.ndarray:
    return cgauss(np.random.default_rng(1000 + level), dim)


def mg_input(dim: int) -> np.ndarray:
    return cgauss(np.random.default_rng(3000), dim)


def elem_samples(ne: int) -> list[int]:
    return sorted({0, 1, ne // 2 + 1, ne - 1, int(np.random.default_rng(7).integers(ne))})


def generate(c: int, nrhs: int = 1, threads: int = 0) -> dict:
    """The fixture arrays of config c (oracle run at full size)."""
    from oracle import pyoracle

    class A:  # argparse-like view for the body below
        pass
    args = A()
    args.rhs, args.threads = nrhs, threads or os.cpu_count() or 1
    t0 = time.time()
    log = lambda msg: print(f"[golden cfg{c} {time.time() - t0:7.1f}s] {msg}", flush=True)  # noqa: E731
    pyoracle.set_lean_elements(True)  # T / H only per element (cfg3: 160 GB otherwise)
    smp = pyoracle.sample(2, c, c)
    n, order = smp["n"], smp["order"]
    ne, nb = n * n, 4 * (order - 1)
    S = pyoracle.Session.from_sample(smp, KAPPA[c], threads=args.threads)
    log(f"elements + skeleton (dim {S.dim}) {S.timings()}")
    out = {}
    wT, rT, wH = elem_vectors(nb)
    sT = np.zeros((ne, 2), dtype=np.complex128)
    sH = np.zeros(ne, dtype=np.complex128)
    nT = np.zeros(ne)
    nH = np.zeros(ne)
    picks = elem_samples(ne)
    Ts, Hs = [], []
    for e in range(ne):
        T, H = S.element(e)
        for p in range(2):
            sT[e, p] = wT[p].conj() @ (T @ rT[p])
        sH[e] = wH.conj() @ H
        nT[e] = np.linalg.norm(T)
        nH[e] = np.linalg.norm(H)
        if e in picks:
            Ts.append(T)
            Hs.append(H)
    out.update(elem_ids=np.array(picks), T_samples=np.array(Ts), H_samples=np.array(Hs),
               sT=sT, sH=sH, nT=nT, nH=nH)
    rhs = S.rhs()
    out.update(q_rhs=sketch(201, rhs), n_rhs=np.linalg.norm(rhs))
    log("element sketches")

    S.build_hierarchy(0, False)
    L = 2 * (n.bit_length() - 1)
    log(f"hierarchy ({L} levels) {S.timings()['hierarchy']:.1f}s")
    q_lv, n_lv = [], []
    for level in range(1, L + 1):
        dim_l = S.level_dim(level)
        y = S.level_apply(level, level_input(level, dim_l))
        q_lv.append(sketch(2000 + level, y))
        n_lv.append(np.linalg.norm(y))
    out.update(q_levels=np.array(q_lv), n_levels=np.array(n_lv))
    log("level sketches")

    S.precond(depth=L, gamma=1, coarse_iters=4)
    z = S.precond_apply(mg_input(S.dim))
    out.update(q_mg=sketch(3001, z), n_mg=np.linalg.norm(z))
    log("MG(v)")

    its, fres, q_x, n_x, hists, q_rhs_b = [], [], [], [], [], []
    for b in range(args.rhs):
        rb = S.rhs() if b == 0 else S.rhs_for(smp["tside"][b])
        x, rep = S.solve(rb, True, restart=RESTART[c], tol=TOL[c], reorth=True,
                         record_history=True)
        its.append(rep["iterations"])
        fres.append(rep["final_residual"])
        q_x.append(sketch(4001, x))
        n_x.append(np.linalg.norm(x))
        q_rhs_b.append(sketch(201, rb))
        h = np.zeros(2000)
        h[:len(rep["residual_history"])] = rep["residual_history"]
        hists.append(h[:max(its[-1], 1)])
        log(f"fgmres rhs {b}: {rep['iterations']} iterations, residual {rep['final_residual']:.3e}")
    out.update(iterations=np.array(its), final_residual=np.array(fres), q_x=np.array(q_x),
               n_x=np.array(n_x), q_rhs_b=np.array(q_rhs_b))
    for b, h in enumerate(hists):
        out[f"history_{b}"] = h
    meta = {"config": c, "seed": c, "n": int(n), "order": int(order), "kappa": KAPPA[c],
            "dim": int(S.dim), "levels": L, "restart": RESTART[c], "tol": TOL[c], "rhs": args.rhs,
            "mg": {"depth": L, "gamma": 1, "coarse_iters": 4}, "reorthogonalize": True,
            "threads": args.threads, "seconds": round(time.time() - t0, 1),
            "generator": "tools/make_golden.py (oracle/ restatement of the reference)"}
    out["meta"] = np.array(json.dumps(meta))
    S.close()
    pyoracle.set_lean_elements(False)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--rhs", type=int, default=1, help="right-hand sides to solve (cfg4: 4)")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    args = ap.parse_args()
    out = generate(args.config, args.rhs, args.threads)
    os.makedirs(args.out, exist_ok=True)
    path = os.path.join(args.out, f"cfg{args.config}.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB)", flush=True)


if __name__ == "__main__":
    main()
