"""Parity of the B200 path (through the C ABI) against the CPU oracle.

Tolerances are BASELINE.json north_star's: ItI and merge operators within
1e-10 relative Frobenius error, final solution within 1e-9 relative L2,
GMRES iteration counts within +-1; integer structure bit-exact (see
tests/test_abi_cpu.py).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_OP = 1e-10
TOL_SOL = 1e-9


def relf(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def hps():
    import paper_2511_00735_b200 as hps
    return hps


@pytest.fixture(scope="module")
def ctx(hps):
    return hps.Context(0)


class Case:
    def __init__(self, hps, oracle, ctx, kind, config, n=0, order=0, kappa=0.0, seed=None,
                 depth=0):
        self.prob = hps.problem(kind, config, seed=seed, n=n, order=order, kappa=kappa)
        p = self.prob
        self.S = oracle.Session(p.n, p.order, p.kappa, p.eta, p.coeff, p.source, p.tside[0])
        self.el = hps.build_elements(ctx, p)
        self.sk = hps.assemble_skeleton(self.el, p)
        self.depth = depth


_cases = {}


def case(hps, oracle, ctx, name):
    if name not in _cases:
        spec = {
            "cfg0": dict(kind=2, config=0),
            "cfg1": dict(kind=2, config=1),
            "bump_n4_N4": dict(kind=0, config=0, n=4, order=4, kappa=6.0),
            "pw_n4_N16": dict(kind=1, config=0, n=4, order=16, kappa=20.0),
            "cfg2_n8": dict(kind=2, config=2, n=8),
            "cfg3_n4": dict(kind=2, config=3, n=4),
            "cfg4_n8": dict(kind=2, config=4, n=8),
        }[name]
        _cases[name] = Case(hps, oracle, ctx, **spec)
    return _cases[name]


ALL = ["cfg0", "bump_n4_N4", "pw_n4_N16", "cfg2_n8", "cfg3_n4", "cfg4_n8", "cfg1"]


@pytest.mark.parametrize("name", ALL)
def test_element_iti_and_source(hps, oracle, ctx, name):
    c = case(hps, oracle, ctx, name)
    T, H = c.el.iti()
    worst_t = worst_h = 0.0
    for e in range(c.prob.n ** 2):
        To, Ho = c.S.element(e)
        worst_t = max(worst_t, relf(T[e], To))
        if np.linalg.norm(Ho) > 0:
            worst_h = max(worst_h, relf(H[e], Ho))
        else:
            assert np.linalg.norm(H[e]) == 0.0  # zero source gives exactly zero H
    assert worst_t < TOL_OP, worst_t
    assert worst_h < TOL_OP, worst_h


@pytest.mark.parametrize("config", [0, 1, 2, 3, 4])
def test_element_cholesky_path_full_configs(hps, oracle, config):
    """At the BASELINE configs' full sizes the interior block is positive
    definite: the batched Cholesky path must handle
    every element with no pivoted-LU fallback launch; sampled elements match
    the oracle's reference-formula element (element.cpp:127-160)."""
    prob = hps.problem(2, config, seed=config)
    fresh = hps.Context(0)
    fresh.profile(True)
    el = hps.build_elements(fresh, prob)
    assert el.fallbacks() == 0
    ne = prob.n ** 2
    picks = sorted({0, ne // 2 + 1, ne - 1})
    for e in picks:
        T, _ = el.iti(e, 1)
        To = oracle.element(prob.order, 1.0 / prob.n, prob.eta, prob.coeff[e])[0]
        assert relf(T[0], To) < TOL_OP, (config, e)


def test_element_indefinite_fallback(hps, oracle, ctx):
    """kappa^2 above the smallest interior eigenvalue (n = 8, N = 8,
    kappa = 41.9): L_ii is indefinite, the device-listed elements take the
    pivoted-LU fallback inside the same (non-blocking) element stage, and the
    maps still match the oracle."""
    prob = hps.problem(1, 0, n=8, order=8, kappa=41.88790204786391)
    el = hps.build_elements(ctx, prob)
    assert el.fallbacks() > 0
    T, _ = el.iti()
    for e in (0, 27, 63):
        To = oracle.element(prob.order, 1.0 / prob.n, prob.eta, prob.coeff[e])[0]
        assert relf(T[e], To) < TOL_OP, e


def test_element_pivoted_inverse_path(hps, oracle, ctx, monkeypatch):
    """The ItI inverses run without pivoting, guarded, with a pivoted redo of
    flagged elements; HPSB_ITI_PIVOT=1 forces the pivoted pass for every
    element.  Both paths give the same maps (and the oracle's)."""
    c = case(hps, oracle, ctx, "cfg1")
    T0, H0 = c.el.iti()
    monkeypatch.setenv("HPSB_ITI_PIVOT", "1")
    el = hps.build_elements(ctx, c.prob)
    T1, H1 = el.iti()
    assert relf(T1, T0) < 1e-12 and relf(H1, H0) < 1e-12
    for e in (0, 77, 255):
        assert relf(T1[e], c.S.element(e)[0]) < TOL_OP


@pytest.mark.parametrize("name", ALL)
def test_skeleton_rhs_and_matvec(hps, oracle, ctx, name):
    c = case(hps, oracle, ctx, name)
    assert c.sk.dim == c.S.dim
    r = c.sk.rhs()
    ro = c.S.rhs()
    if np.linalg.norm(ro) == 0:
        assert np.linalg.norm(r) == 0
    else:
        assert relf(r, ro) < TOL_OP
    rng = np.random.default_rng(11)
    x = rng.standard_normal(c.sk.dim) + 1j * rng.standard_normal(c.sk.dim)
    assert relf(c.sk.apply(x), c.S.apply_M(x)) < TOL_OP


@pytest.mark.parametrize("name", ["cfg0", "pw_n4_N16", "cfg4_n8"])
def test_skeleton_boundary_layout_matches_element_layout(hps, oracle, ctx, name):
    """hpsb_skeleton_create_boundary (physical sides only) and
    hpsb_skeleton_create (element-side layout) give bit-identical right-hand
    sides and recovered fields for every right-hand side."""
    c = case(hps, oracle, ctx, name)
    sk_full = hps.assemble_skeleton(c.el, c.prob, boundary_only=False)
    assert sk_full.nrhs == c.sk.nrhs == c.prob.tside.shape[0]
    for r in range(c.sk.nrhs):
        assert np.array_equal(c.sk.rhs(r), sk_full.rhs(r))
    rng = np.random.default_rng(5)
    g = rng.standard_normal(c.sk.dim) + 1j * rng.standard_normal(c.sk.dim)
    assert np.array_equal(c.sk.recover(g, c.sk.nrhs - 1), sk_full.recover(g, c.sk.nrhs - 1))


MERGE_MODES = {
    "diag": {},                                  # default: diagonal pivots, guarded
    "pivot": {"HPSB_MERGE_PIVOT": "1"},          # partial pivoting throughout
    "redo": {"HPSB_TEST_GUARD_TRIP": "1"},       # guard tripped: pivoted rebuild
}


@pytest.mark.parametrize("mode", list(MERGE_MODES))
@pytest.mark.parametrize("name", ["cfg0", "bump_n4_N4", "cfg3_n4", "cfg2_n8", "cfg1"])
def test_hierarchy_level_systems(hps, oracle, ctx, name, mode, monkeypatch):
    """Every level system M_l within 1e-10 of the oracle's, for the merge
    inverses on diagonal pivots (default; cfg1 / cfg2_n8 reach the blocked
    path with s = 120), with partial pivoting, and through the pivoted
    rebuild that a tripped guard takes."""
    for k, v in MERGE_MODES[mode].items():
        monkeypatch.setenv(k, v)
    c = case(hps, oracle, ctx, name)
    h = hps.build_hierarchy(c.sk)
    c.S.build_hierarchy(0, True)
    bs = 2 * c.el.m
    for level in range(1, h.depth + 1):
        ff, blocks = h.level_blocks(level)
        ffo, bo = c.S.level_blocks(level)
        assert ff == ffo
        nf = 2 * c.prob.n * (c.prob.n - 1) - ff
        A = np.zeros((nf * bs, nf * bs), dtype=complex)
        B = np.zeros_like(A)
        for (r, cc), b in blocks.items():
            A[r * bs:(r + 1) * bs, cc * bs:(cc + 1) * bs] = b
        for (r, cc), b in bo.items():
            B[r * bs:(r + 1) * bs, cc * bs:(cc + 1) * bs] = b
        assert relf(A, B) < TOL_OP, (level, relf(A, B))


def test_n4_block_sparsity_patterns(hps, oracle, ctx):
    # test_dissection.cpp:365-433 on the GPU hierarchy
    c = case(hps, oracle, ctx, "bump_n4_N4")
    h = hps.build_hierarchy(c.sk)
    M2 = {0: [0, 1, 8, 9, 12, 13], 8: [0, 1, 4, 5, 8], 9: [0, 1, 4, 5, 9, 12, 13, 14, 15],
          12: [0, 1, 2, 3, 9, 10, 12, 13]}
    _, blocks = h.level_blocks(2)
    scale = max(np.abs(b).max() for b in blocks.values())
    for r, cols in M2.items():
        got = sorted(cc for (rr, cc), b in blocks.items() if rr == r and np.abs(b).max() > 1e-12 * scale)
        assert got == cols, (r, got)


def test_merge_pair(hps, oracle, ctx):
    c = case(hps, oracle, ctx, "cfg0")
    g = hps.face_graph(c.prob.n)
    for f in (0, 8, 16):
        e1, e2, s1, s2 = (int(v) for v in g["faces"][f][:4])
        T1, H1 = c.S.element(e1)
        T2, H2 = c.S.element(e2)
        To, Ho = oracle.merge_pair(T1, H1, T2, H2, s1, s2, c.el.m)
        Tg, Hg = hps.merge_pair(ctx, T1, H1, T2, H2, s1, s2, c.el.m)
        assert relf(Tg, To) < TOL_OP
        assert relf(Hg, Ho) < TOL_OP


@pytest.mark.parametrize("name", ["cfg0", "bump_n4_N4", "cfg3_n4", "cfg2_n8", "cfg1"])
def test_preconditioner_apply(hps, oracle, ctx, name):
    c = case(hps, oracle, ctx, name)
    h = hps.build_hierarchy(c.sk)
    c.S.build_hierarchy(0, False)
    pc = hps.build_preconditioner(h, coarse_iters=4)
    c.S.precond(depth=h.depth, gamma=1, coarse_iters=4)
    rng = np.random.default_rng(5)
    for _ in range(3):
        v = rng.standard_normal(c.sk.dim) + 1j * rng.standard_normal(c.sk.dim)
        assert relf(pc.apply(v), c.S.precond_apply(v)) < TOL_OP


@pytest.mark.parametrize("name", ["cfg0", "bump_n4_N4", "pw_n4_N16", "cfg1"])
def test_fgmres_solution_and_iterations(hps, oracle, ctx, name):
    c = case(hps, oracle, ctx, name)
    h = hps.build_hierarchy(c.sk)
    c.S.build_hierarchy(0, False)
    pc = hps.build_preconditioner(h, coarse_iters=4)
    c.S.precond(depth=h.depth, gamma=1, coarse_iters=4)
    rhs = c.sk.rhs()
    x, rep = hps.fgmres(c.sk, rhs, pc, restart=c.prob.restart, tol=c.prob.tol)
    xo, repo = c.S.solve(c.S.rhs(), True, restart=c.prob.restart, tol=c.prob.tol)
    assert rep["converged"] and repo["converged"]
    assert abs(rep["iterations"] - repo["iterations"]) <= 1, (rep, repo)
    assert relf(x, xo) < TOL_SOL


@pytest.mark.parametrize("name", ["cfg0", "cfg1", "bump_n4_N4"])
def test_fgmres_device_cycle_graph(hps, oracle, ctx, name, monkeypatch):
    """The device-driven restart cycle (HPSB_CYCLE_GRAPH=1: Arnoldi steps and
    Givens updates in a CUDA graph WHILE node) ends where the host loop does
    (krylov.cpp:92-123) and matches the oracle; unpreconditioned too, and
    with small restarts (several cycles) and the residual history."""
    c = case(hps, oracle, ctx, name)
    h = hps.build_hierarchy(c.sk)
    pc = hps.build_preconditioner(h, coarse_iters=4)
    rhs = c.sk.rhs()
    x0, rep0 = hps.fgmres(c.sk, rhs, pc, restart=c.prob.restart, tol=c.prob.tol)
    xs, reps = hps.fgmres(c.sk, rhs, pc, restart=5, tol=c.prob.tol, record_history=True)
    xu, repu = hps.fgmres(c.sk, rhs, None, restart=30, tol=1e-8, max_iters=60)
    monkeypatch.setenv("HPSB_CYCLE_GRAPH", "1")
    x1, rep1 = hps.fgmres(c.sk, rhs, pc, restart=c.prob.restart, tol=c.prob.tol)
    xs1, reps1 = hps.fgmres(c.sk, rhs, pc, restart=5, tol=c.prob.tol, record_history=True)
    xu1, repu1 = hps.fgmres(c.sk, rhs, None, restart=30, tol=1e-8, max_iters=60)
    assert rep1["converged"] and reps1["converged"]
    assert repu1["iterations"] == repu["iterations"] and relf(xu1, xu) < 1e-12
    h0, h1 = np.asarray(reps["residual_history"]), np.asarray(reps1["residual_history"])
    assert h0.shape == h1.shape and np.allclose(h0, h1, rtol=1e-5, atol=0)  # estimates near 1e-10: rounding
    assert rep1["iterations"] == rep0["iterations"] and reps1["iterations"] == reps["iterations"]
    assert relf(x1, x0) < 1e-12 and relf(xs1, xs) < 1e-12
    c.S.build_hierarchy(0, False)
    c.S.precond(depth=h.depth, gamma=1, coarse_iters=4)
    xo, repo = c.S.solve(c.S.rhs(), True, restart=c.prob.restart, tol=c.prob.tol)
    assert abs(rep1["iterations"] - repo["iterations"]) <= 1 and relf(x1, xo) < TOL_SOL


@pytest.mark.parametrize("name", ["cfg3_n4", "cfg2_n8", "cfg4_n8"])
def test_fgmres_underresolved_meshes(hps, oracle, ctx, name):
    # The configs' wavenumbers on 4x4 / 8x8 meshes (kappa h up to 100) give
    # systems needing ~100 iterations.  The preconditioner contains an inner
    # GMRES, so it is a nonlinear function of its input: last-bit differences
    # (CGS2 vs MGS, summation order) grow ~2x per iteration (measured: 1e-15
    # at step 1, 1e-12 at step 11) and the count wanders by up to ~20%.  These
    # shrunken meshes (not BASELINE configs) therefore pin the converged
    # solution and residual, with a loose bound on the count.
    c = case(hps, oracle, ctx, name)
    h = hps.build_hierarchy(c.sk)
    c.S.build_hierarchy(0, False)
    pc = hps.build_preconditioner(h, coarse_iters=4)
    c.S.precond(depth=h.depth, gamma=1, coarse_iters=4)
    x, rep = hps.fgmres(c.sk, c.sk.rhs(), pc, restart=100, tol=1e-10)
    xo, repo = c.S.solve(c.S.rhs(), True, restart=100, tol=1e-10)
    assert rep["converged"] and repo["converged"]
    assert abs(rep["iterations"] - repo["iterations"]) <= max(1, repo["iterations"] // 4)
    assert relf(x, xo) < 1e-8
    r = c.S.rhs() - c.S.apply_M(x)
    assert np.linalg.norm(r) <= 1e-10 * np.linalg.norm(c.S.rhs()) * 1.01


def test_unpreconditioned_gmres(hps, oracle, ctx):
    c = case(hps, oracle, ctx, "cfg0")
    x, rep = hps.gmres(c.sk, c.sk.rhs(), restart=50, tol=1e-10)
    xo, repo = c.S.solve(c.S.rhs(), False, restart=50, tol=1e-10)
    assert rep["converged"]
    assert abs(rep["iterations"] - repo["iterations"]) <= 1
    assert relf(x, xo) < TOL_SOL


def _planewave_field_l2(oracle, n, order, kappa, field):
    """Mass-weighted relative L2 error of a recovered field against exp(i kappa x)
    (test_problems.cpp:65-71's plane-wave accuracy check)."""
    x, w, _ = oracle.gll_rule(order)
    s = oracle.index_sets(order)
    np1, h = order + 1, 1.0 / n
    ii, jj = s["noncorner"] // np1, s["noncorner"] % np1
    err2 = ref2 = 0.0
    for e in range(n * n):
        X = h * (e % n) + 0.5 * (x[ii] + 1) * h
        ref = np.exp(1j * kappa * X)
        wt = (0.5 * h * w[ii]) * (0.5 * h * w[jj])
        err2 += np.sum(wt * np.abs(field[e] - ref) ** 2)
        ref2 += np.sum(wt * np.abs(ref) ** 2)
    return np.sqrt(err2 / ref2)


@pytest.mark.parametrize("name", ALL)
def test_recover_field(hps, oracle, ctx, name):
    # recover_solution (problems.cpp:60-92) on the same skeleton data.
    c = case(hps, oracle, ctx, name)
    rng = np.random.default_rng(7)
    g = rng.standard_normal(c.sk.dim) + 1j * rng.standard_normal(c.sk.dim)
    f = c.sk.recover(g)
    fo = c.S.recover(g)
    assert f.shape == fo.shape
    assert relf(f, fo) < TOL_OP


def test_recover_planewave_after_fgmres(hps, oracle, ctx):
    # End to end on the GPU: rhs -> FGMRES -> field, against the exact plane
    # wave (test_problems.cpp:65-71, <= 1e-8) and the oracle's field (1e-9).
    c = case(hps, oracle, ctx, "pw_n4_N16")
    h = hps.build_hierarchy(c.sk)
    pc = hps.build_preconditioner(h, coarse_iters=4)
    x, rep = hps.fgmres(c.sk, c.sk.rhs(), pc, restart=50, tol=1e-12)
    assert rep["converged"]
    f = c.sk.recover(x)
    assert _planewave_field_l2(oracle, c.prob.n, c.prob.order, c.prob.kappa, f) < 1e-8
    c.S.build_hierarchy(0, True)
    fo = c.S.recover(c.S.direct_solve(c.S.rhs()))
    assert relf(f, fo) < TOL_SOL


@pytest.mark.parametrize("name", ["cfg0", "bump_n4_N4", "cfg2_n8", "cfg1"])
def test_direct_solve(hps, oracle, ctx, name):
    # direct_solve (dissection.cpp:240-292) against the oracle's, and the
    # residual of the dense-coarse block elimination.
    c = case(hps, oracle, ctx, name)
    h = hps.build_hierarchy(c.sk, factor_coarse=True)
    c.S.build_hierarchy(0, True)
    rhs = c.sk.rhs()
    x = h.direct_solve(rhs)
    xo = c.S.direct_solve(c.S.rhs())
    assert relf(x, xo) < TOL_SOL
    assert np.linalg.norm(rhs - c.S.apply_M(x)) < 1e-9 * np.linalg.norm(rhs)


def test_direct_solve_needs_factored_full_depth(hps, oracle, ctx):
    c = case(hps, oracle, ctx, "cfg0")
    h = hps.build_hierarchy(c.sk, factor_coarse=False)
    with pytest.raises(hps.HpsError, match="full depth"):
        h.direct_solve(c.sk.rhs())
    h2 = hps.build_hierarchy(c.sk, depth=2, factor_coarse=True)
    with pytest.raises(hps.HpsError, match="full depth"):
        h2.direct_solve(c.sk.rhs())


@pytest.mark.parametrize("name", ["cfg0", "bump_n4_N4", "cfg2_n8", "cfg1"])
def test_exact_coarse_full_depth(hps, oracle, ctx, name):
    # MgConfig.exact_coarse (multigrid.cpp:22-27, :37-38) at full depth: the
    # V-cycle is an exact inverse, so FGMRES converges in one iteration.
    c = case(hps, oracle, ctx, name)
    h = hps.build_hierarchy(c.sk, factor_coarse=False)
    c.S.build_hierarchy(0, True)
    pc = hps.build_preconditioner(h, exact_coarse=True)
    c.S.precond(depth=h.depth, gamma=1, coarse_iters=4, exact=True)
    rng = np.random.default_rng(11)
    v = rng.standard_normal(c.sk.dim) + 1j * rng.standard_normal(c.sk.dim)
    assert relf(pc.apply(v), c.S.precond_apply(v)) < TOL_OP
    x, rep = hps.fgmres(c.sk, c.sk.rhs(), pc, restart=10, tol=1e-10)
    assert rep["converged"] and rep["iterations"] <= 2, rep
    assert relf(x, c.S.direct_solve(c.S.rhs())) < TOL_SOL


@pytest.mark.parametrize("name", ["cfg0", "bump_n4_N4", "cfg2_n8"])
def test_exact_coarse_partial_depth(hps, oracle, ctx, name):
    c = case(hps, oracle, ctx, name)
    h = hps.build_hierarchy(c.sk, depth=2, factor_coarse=False)
    c.S.build_hierarchy(0, False)
    pc = hps.build_preconditioner(h, exact_coarse=True)
    c.S.precond(depth=2, gamma=1, coarse_iters=4, exact=True)
    rng = np.random.default_rng(12)
    v = rng.standard_normal(c.sk.dim) + 1j * rng.standard_normal(c.sk.dim)
    assert relf(pc.apply(v), c.S.precond_apply(v)) < TOL_OP
    x, rep = hps.fgmres(c.sk, c.sk.rhs(), pc, restart=50, tol=1e-10)
    xo, repo = c.S.solve(c.S.rhs(), True, restart=50, tol=1e-10)
    assert rep["converged"] and abs(rep["iterations"] - repo["iterations"]) <= 1, (rep, repo)
    assert relf(x, xo) < TOL_SOL


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.float64)).cuda()


def test_multi_rhs_operators(hps, oracle, ctx):
    # Multi-RHS interface matvec and MG apply (one pass over the maps for R
    # vectors, DMMA GEMMs) against the single-RHS path column by column.
    import torch
    c = case(hps, oracle, ctx, "cfg2_n8")
    h = hps.build_hierarchy(c.sk, factor_coarse=False)
    pc = hps.build_preconditioner(h, coarse_iters=4)
    R = 5
    rng = np.random.default_rng(21)
    X = rng.standard_normal((R, c.sk.dim)) + 1j * rng.standard_normal((R, c.sk.dim))
    xd = _dev(torch, X)
    yd = torch.empty_like(xd)
    hps._check(hps._lib.hpsb_skeleton_apply_batch_dev(c.sk._h, xd.data_ptr(), yd.data_ptr(), R))
    ctx.synchronize()  # the library stream is not torch's
    Y = yd.cpu().numpy().view(np.complex128).reshape(R, -1)
    for b in range(R):
        assert relf(Y[b], c.sk.apply(X[b])) < 1e-13
    zd = torch.empty_like(xd)
    hps._check(hps._lib.hpsb_precond_apply_batch_dev(pc._h, xd.data_ptr(), zd.data_ptr(), R))
    ctx.synchronize()
    Z = zd.cpu().numpy().view(np.complex128).reshape(R, -1)
    for b in range(R):
        assert relf(Z[b], pc.apply(X[b])) < TOL_OP


@pytest.mark.parametrize("exact", [False, True])
def test_multi_rhs_precond_exact_and_partial(hps, oracle, ctx, exact):
    import torch
    c = case(hps, oracle, ctx, "bump_n4_N4")
    h = hps.build_hierarchy(c.sk, factor_coarse=False)
    pc = hps.build_preconditioner(h, coarse_iters=3, exact_coarse=exact)
    R = 3
    rng = np.random.default_rng(22)
    X = rng.standard_normal((R, c.sk.dim)) + 1j * rng.standard_normal((R, c.sk.dim))
    xd = _dev(torch, X)
    zd = torch.empty_like(xd)
    hps._check(hps._lib.hpsb_precond_apply_batch_dev(pc._h, xd.data_ptr(), zd.data_ptr(), R))
    ctx.synchronize()
    Z = zd.cpu().numpy().view(np.complex128).reshape(R, -1)
    for b in range(R):
        assert relf(Z[b], pc.apply(X[b])) < TOL_OP


def test_fgmres_multi_rhs_cfg4_planewaves(hps, oracle, ctx):
    # cfg4's setting (32 plane-wave right-hand sides, s = 0) on an 8 x 8 mesh:
    # R right-hand sides in lockstep, each against its own oracle solve.
    p = hps.problem(2, 4, n=8)
    el = hps.build_elements(ctx, p)
    sk = hps.assemble_skeleton(el, p)
    h = hps.build_hierarchy(sk, factor_coarse=False)
    pc = hps.build_preconditioner(h, coarse_iters=4)
    R = 4
    rhs = np.stack([sk.rhs(b) for b in range(R)])
    X, reps = hps.fgmres_batch(sk, rhs, pc, restart=100, tol=1e-10)
    for b in range(R):
        S = oracle.Session(p.n, p.order, p.kappa, p.eta, p.coeff, p.source, p.tside[b])
        assert relf(rhs[b], S.rhs()) < TOL_OP
        S.build_hierarchy(0, False)
        S.precond(depth=h.depth, gamma=1, coarse_iters=4)
        xo, repo = S.solve(S.rhs(), True, restart=100, tol=1e-10)
        assert reps[b]["converged"] and repo["converged"]
        assert abs(reps[b]["iterations"] - repo["iterations"]) <= max(1, repo["iterations"] // 4)
        assert relf(X[b], xo) < 1e-8
        # and exactly the single-RHS GPU solve's iteration count
        xs, reps1 = hps.fgmres(sk, rhs[b], pc, restart=100, tol=1e-10)
        assert abs(reps1["iterations"] - reps[b]["iterations"]) <= 1
        assert relf(X[b], xs) < TOL_SOL


@pytest.mark.parametrize("name", ["cfg0", "bump_n4_N4", "cfg2_n8"])
@pytest.mark.parametrize("gamma", [2, 3])
def test_gamma_cycle(hps, oracle, ctx, name, gamma):
    # apply_level's gamma recursion (multigrid.cpp:71-80): gamma coarse
    # corrections per level with the level-system residual in between.
    c = case(hps, oracle, ctx, name)
    h = hps.build_hierarchy(c.sk, factor_coarse=False)
    c.S.build_hierarchy(0, False)
    pc = hps.build_preconditioner(h, gamma=gamma, coarse_iters=4)
    c.S.precond(depth=h.depth, gamma=gamma, coarse_iters=4)
    rng = np.random.default_rng(30 + gamma)
    v = rng.standard_normal(c.sk.dim) + 1j * rng.standard_normal(c.sk.dim)
    assert relf(pc.apply(v), c.S.precond_apply(v)) < TOL_OP
    if name != "cfg2_n8":
        x, rep = hps.fgmres(c.sk, c.sk.rhs(), pc, restart=50, tol=1e-10)
        xo, repo = c.S.solve(c.S.rhs(), True, restart=50, tol=1e-10)
        assert rep["converged"] and abs(rep["iterations"] - repo["iterations"]) <= 1
        assert relf(x, xo) < TOL_SOL
