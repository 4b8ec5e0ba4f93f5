"""The reference entry points' semantics at the C-ABI boundary, against the oracle.

- a preconditioner shallower than its hierarchy (MgConfig{depth} <
  build_hierarchy depth; multigrid.cpp:13-16,24-26 -- the reference default
  MgConfig{} has depth 2, multigrid.hpp:13);
- KrylovConfig.reorthogonalize = false: one modified Gram-Schmidt pass
  (krylov.cpp:98-102, the KrylovConfig default, krylov.hpp:19);
- gmres with a fixed right preconditioner (krylov.cpp:180-186);
- SolveReport's basis_orthogonality / precond_memory / wall_build
  (krylov.hpp:23-34; test_driver.cpp:70-117 contracts);
- restart > 100, coarse_iters > 60, gamma > 16 (no B200-only limits);
- several contexts on one host thread (per-context allocation streams).
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


_cache = {}


def setup(hps, oracle, ctx, name):
    if name not in _cache:
        spec = {"cfg0": dict(kind=2, config=0), "cfg1": dict(kind=2, config=1),
                "bump": dict(kind=0, config=0, n=4, order=4, kappa=6.0)}[name]
        p = hps.problem(**spec)
        S = oracle.Session(p.n, p.order, p.kappa, p.eta, p.coeff, p.source, p.tside[0])
        el = hps.build_elements(ctx, p)
        sk = hps.assemble_skeleton(el, p)
        h = hps.build_hierarchy(sk, factor_coarse=False)
        S.build_hierarchy(0, False)
        _cache[name] = (p, S, el, sk, h)
    return _cache[name]


@pytest.mark.parametrize("name", ["cfg0", "cfg1"])
@pytest.mark.parametrize("depth", [2, 3])
def test_precond_shallower_than_hierarchy(hps, oracle, ctx, name, depth):
    p, S, el, sk, h = setup(hps, oracle, ctx, name)
    assert h.depth > depth
    pc = hps.build_preconditioner(h, depth=depth, coarse_iters=4)
    S.precond(depth=depth, gamma=1, coarse_iters=4)
    rng = np.random.default_rng(40 + depth)
    v = rng.standard_normal(sk.dim) + 1j * rng.standard_normal(sk.dim)
    assert relf(pc.apply(v), S.precond_apply(v)) < TOL_OP
    x, rep = hps.fgmres(sk, sk.rhs(), pc, restart=p.restart, tol=p.tol)
    xo, repo = S.solve(S.rhs(), True, restart=p.restart, tol=p.tol)
    assert rep["converged"] and abs(rep["iterations"] - repo["iterations"]) <= 1, (rep, repo)
    assert relf(x, xo) < TOL_SOL


@pytest.mark.parametrize("name", ["cfg0", "cfg1", "bump"])
def test_single_pass_mgs(hps, oracle, ctx, name):
    """reorthogonalize = false: the reference's single MGS pass, preconditioned
    and not."""
    p, S, el, sk, h = setup(hps, oracle, ctx, name)
    pc = hps.build_preconditioner(h, coarse_iters=4)
    S.precond(depth=h.depth, gamma=1, coarse_iters=4)
    x, rep = hps.fgmres(sk, sk.rhs(), pc, restart=p.restart, tol=1e-10, reorthogonalize=False)
    xo, repo = S.solve(S.rhs(), True, restart=p.restart, tol=1e-10, reorth=False)
    assert rep["converged"] and abs(rep["iterations"] - repo["iterations"]) <= 1, (rep, repo)
    assert relf(x, xo) < TOL_SOL
    xu, repu = hps.gmres(sk, sk.rhs(), restart=30, tol=1e-8, max_iters=90, reorthogonalize=False)
    xuo, repuo = S.solve(S.rhs(), False, restart=30, tol=1e-8, max_iters=90, reorth=False)
    assert abs(repu["iterations"] - repuo["iterations"]) <= 1, (repu, repuo)
    if repuo["converged"]:
        assert relf(xu, xuo) < 1e-7


@pytest.mark.parametrize("name", ["cfg0", "cfg1"])
@pytest.mark.parametrize("reorth", [True, False])
def test_right_preconditioned_gmres(hps, oracle, ctx, name, reorth):
    p, S, el, sk, h = setup(hps, oracle, ctx, name)
    pc = hps.build_preconditioner(h, coarse_iters=4)
    S.precond(depth=h.depth, gamma=1, coarse_iters=4)
    x, rep = hps.gmres(sk, sk.rhs(), restart=p.restart, tol=1e-10, right_precond=pc,
                       reorthogonalize=reorth)
    xo, repo = S.solve(S.rhs(), "right", restart=p.restart, tol=1e-10, reorth=reorth)
    assert rep["converged"] and repo["converged"]
    assert abs(rep["iterations"] - repo["iterations"]) <= 1, (rep, repo)
    assert relf(x, xo) < TOL_SOL


def test_solve_report_fields(hps, oracle, ctx):
    """test_driver.cpp:70-117: basis orthogonality <= 1e-8 with
    record_history on the driver's reorthogonalised solve, a positive
    preconditioner memory, build / solve times.  A single MGS pass (the
    KrylovConfig default) keeps the basis orthogonal only to ~1e-6 here, on
    the oracle as on the GPU."""
    p, S, el, sk, h = setup(hps, oracle, ctx, "cfg1")
    pc = hps.build_preconditioner(h, depth=3, coarse_iters=4)
    S.precond(depth=3, gamma=1, coarse_iters=4)
    for reorth in (True, False):
        x, rep = hps.fgmres(sk, sk.rhs(), pc, restart=p.restart, tol=p.tol, record_history=True,
                            reorthogonalize=reorth)
        _, repo = S.solve(S.rhs(), True, restart=p.restart, tol=p.tol, record_history=True,
                          reorth=reorth)
        assert rep["converged"]
        if reorth:
            assert 0.0 < rep["basis_orthogonality"] <= 1e-8, rep
            assert repo["basis_orthogonality"] <= 1e-8
        else:
            assert 0.0 < rep["basis_orthogonality"] <= 10 * repo["basis_orthogonality"], (rep, repo)
        assert rep["precond_memory"] > 0 and rep["wall_build"] > 0
        assert rep["wall_solve"] == rep["seconds"] > 0
        assert len(rep["residual_history"]) == rep["iterations"]


@pytest.mark.parametrize("reorth", [True, False])
def test_restart_above_100(hps, oracle, ctx, reorth):
    """restart 150 > the 96 columns one orthogonalisation launch holds:
    150 unpreconditioned Arnoldi steps in one cycle on cfg1 (not converged
    yet), the same iterate as the oracle's."""
    p, S, el, sk, h = setup(hps, oracle, ctx, "cfg1")
    x, rep = hps.gmres(sk, sk.rhs(), restart=150, tol=1e-12, max_iters=150,
                       reorthogonalize=reorth, record_history=True)
    xo, repo = S.solve(S.rhs(), False, restart=150, tol=1e-12, max_iters=150, reorth=reorth,
                       record_history=True)
    assert rep["iterations"] == repo["iterations"] == 150
    assert not rep["converged"] and not repo["converged"]
    assert abs(rep["final_residual"] / repo["final_residual"] - 1) < 1e-6
    h, ho = np.asarray(rep["residual_history"]), np.asarray(repo["residual_history"])
    assert np.allclose(h, ho, rtol=1e-6, atol=0)
    assert relf(x, xo) < 1e-8


def test_coarse_iters_above_60_and_gamma_above_16(hps, oracle, ctx):
    p, S, el, sk, h = setup(hps, oracle, ctx, "cfg1")
    pc = hps.build_preconditioner(h, coarse_iters=70)
    S.precond(depth=h.depth, gamma=1, coarse_iters=70)
    rng = np.random.default_rng(77)
    v = rng.standard_normal(sk.dim) + 1j * rng.standard_normal(sk.dim)
    assert relf(pc.apply(v), S.precond_apply(v)) < TOL_OP
    p0, S0, el0, sk0, h0 = setup(hps, oracle, ctx, "cfg0")
    pg = hps.build_preconditioner(h0, depth=3, gamma=17, coarse_iters=2)
    S0.precond(depth=3, gamma=17, coarse_iters=2)
    v0 = rng.standard_normal(sk0.dim) + 1j * rng.standard_normal(sk0.dim)
    assert relf(pg.apply(v0), S0.precond_apply(v0)) < TOL_OP


def test_two_contexts_on_one_thread(hps, oracle):
    """Objects of two contexts interleaved on one host thread: each context's
    device memory is allocated and released on its own stream (a stage still
    running on one context is unaffected by the other's frees)."""
    pa = hps.problem(2, 1)
    pb = hps.problem(2, 0)
    ca, cb = hps.Context(0), hps.Context(0)
    ela = hps.build_elements(ca, pa)          # enqueued, not waited for
    elb = hps.build_elements(cb, pb)
    ska = hps.assemble_skeleton(ela, pa)
    skb = hps.assemble_skeleton(elb, pb)
    hb = hps.build_hierarchy(skb, factor_coarse=False)
    hb.close(), skb.close(), elb.close()       # B's frees while A may still run
    ha = hps.build_hierarchy(ska, factor_coarse=False)
    pca = hps.build_preconditioner(ha, coarse_iters=4)
    x, rep = hps.fgmres(ska, ska.rhs(), pca, restart=pa.restart, tol=pa.tol)
    S = oracle.Session(pa.n, pa.order, pa.kappa, pa.eta, pa.coeff, pa.source, pa.tside[0])
    S.build_hierarchy(0, False)
    S.precond(depth=ha.depth, gamma=1, coarse_iters=4)
    xo, repo = S.solve(S.rhs(), True, restart=pa.restart, tol=pa.tol)
    assert abs(rep["iterations"] - repo["iterations"]) <= 1
    assert relf(x, xo) < TOL_SOL
    pca.close(), ha.close(), ska.close(), ela.close()
    ca.close(), cb.close()


def test_multi_rhs_single_pass_mgs(hps, oracle, ctx):
    p, S, el, sk, h = setup(hps, oracle, ctx, "cfg0")
    pc = hps.build_preconditioner(h, coarse_iters=4)
    rhs = np.stack([sk.rhs(), 1j * sk.rhs()])
    X, reps = hps.fgmres_batch(sk, rhs, pc, restart=50, tol=1e-10, reorthogonalize=False)
    x1, rep1 = hps.fgmres(sk, sk.rhs(), pc, restart=50, tol=1e-10, reorthogonalize=False)
    for b in range(2):
        assert reps[b]["converged"] and abs(reps[b]["iterations"] - rep1["iterations"]) <= 1
    assert relf(X[0], x1) < TOL_SOL and relf(X[1], 1j * x1) < TOL_SOL
