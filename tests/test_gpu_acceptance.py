"""Table-1 acceptance on the GPU sweep driver, restating
proj/tests/acceptance.cpp:205-291: the desk problem (bump, 16x16 elements,
degree 8, ppw 9.6, tol 1e-8, driver.cpp's fgmres) swept over depth 2..8 and
coarse_iters 4..6, with iteration counts

  * non-increasing in depth (+1 slack) and in coarse_iters (+1 slack),
  * every cell below the unpreconditioned GMRES count,
  * gamma=2/ci=2 within +2 of gamma=1/ci=4 for depth >= 3,

plus a per-cell comparison of the GPU iteration counts with the oracle's on
the same problem (north_star: iterations within +-1)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DEPTHS = list(range(2, 9))


def desk_base(d):  # acceptance.cpp:205-215
    return d.RunConfig(problem="bump", elements=16, degree=8, ppw=9.6, tol=1e-8, mode="mg",
                       record_history=False)


@pytest.fixture(scope="module")
def sweep():
    import paper_2511_00735_b200 as hps
    from paper_2511_00735_b200 import driver as d
    ctx = hps.Context(0)
    base = desk_base(d)
    g1 = d.run_sweep(base, d.SweepAxes(depths=DEPTHS, gammas=[1], coarse_iters=[4, 5, 6]), ctx)
    g2 = d.run_sweep(base, d.SweepAxes(depths=DEPTHS, gammas=[2], coarse_iters=[2]), ctx)
    unprec = d.run_experiment(d.RunConfig(**{**base.__dict__, "mode": "unpreconditioned"}), ctx)
    return g1, g2, unprec


def _iters(cells, depth, gamma, ci):  # acceptance.cpp:217-223
    for c in cells:
        if c.levels == depth and c.gamma == gamma and c.coarse_iters == ci:
            return c.report.iterations if c.converged else -1
    return -1


def test_iteration_trends(sweep):  # acceptance.cpp:225-262
    g1, _, unprec = sweep
    assert unprec.report.converged
    base_its = unprec.report.iterations
    table = {ci: [_iters(g1, dd, 1, ci) for dd in DEPTHS] for ci in (4, 5, 6)}
    for ci, row in table.items():
        prev = 1 << 30
        for dd, its in zip(DEPTHS, row):
            assert its > 0, (ci, dd, table)
            assert its <= prev + 1, ("non-increasing in depth", ci, table)
            assert its < base_its, ("below unpreconditioned", base_its, table)
            prev = its
    for k, dd in enumerate(DEPTHS):
        prev = 1 << 30
        for ci in (4, 5, 6):
            its = table[ci][k]
            assert its <= prev + 1, ("non-increasing in coarse_iters", dd, table)
            prev = its


def test_gamma_cycle_vs_v_cycle(sweep):  # acceptance.cpp:264-291
    g1, g2, _ = sweep
    for dd in DEPTHS:
        two, one = _iters(g2, dd, 2, 2), _iters(g1, dd, 1, 4)
        if dd == 2:
            continue  # informational in the reference
        assert two > 0 and one > 0 and two <= one + 2, (dd, two, one)


@pytest.mark.parametrize("depth,gamma,ci", [(2, 1, 4), (4, 1, 5), (6, 1, 6), (8, 1, 4),
                                            (5, 2, 2), (8, 2, 2)])
def test_sweep_cells_match_oracle(sweep, depth, gamma, ci):
    """The GPU sweep cell's iteration count against the oracle's FGMRES on the
    same problem, hierarchy depth and cycle (driver.cpp:196-261 per cell)."""
    import paper_2511_00735_b200 as hps
    from paper_2511_00735_b200 import driver as d
    from oracle import pyoracle
    g1, g2, _ = sweep
    gpu_its = _iters(g1 if gamma == 1 else g2, depth, gamma, ci)
    base = desk_base(d)
    kappa = d.validate_config(d.RunConfig(**{**base.__dict__, "depth": 0}))
    prob = hps.problem(0, 0, n=base.elements, order=base.degree, kappa=kappa)
    S = pyoracle.Session(prob.n, prob.order, prob.kappa, prob.eta, prob.coeff, prob.source,
                         prob.tside[0])
    S.build_hierarchy(depth, False)
    S.precond(depth=depth, gamma=gamma, coarse_iters=ci)
    _, rep = S.solve(S.rhs(), True, restart=base.restart, tol=base.tol, max_iters=base.max_iters)
    assert rep["converged"]
    assert abs(gpu_its - rep["iterations"]) <= 1, (gpu_its, rep["iterations"])
    assert np.isfinite(rep["final_residual"])
