"""The sharded (quadtree-subtree, multi-rank) path on one GPU.

Ranks are emulated in one process (hpsb_local_group: one host thread and one
context per rank, host barriers for the collectives -- no kernel ever waits
on another rank's kernel).  Every rank must reproduce the single-GPU results:
rhs, matvec, preconditioner apply, FGMRES solution and iteration count.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def relf(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _single(hps, prob, x, v):
    ctx = hps.Context(0)
    el = hps.build_elements(ctx, prob)
    sk = hps.assemble_skeleton(el, prob)
    h = hps.build_hierarchy(sk)
    pc = hps.build_preconditioner(h, coarse_iters=4)
    sol, rep = hps.fgmres(sk, sk.rhs(), pc, restart=prob.restart, tol=prob.tol)
    pe = hps.build_preconditioner(h, exact_coarse=True)
    return {"rhs": sk.rhs(), "Mx": sk.apply(x), "Pv": pc.apply(v), "x": sol, "rep": rep,
            "Pe": pe.apply(v), "direct": h.direct_solve(sk.rhs()), "field": sk.recover(sol)}


def _sharded(hps, prob, world, x, v):
    grp = hps.LocalGroup(world)
    out, errs = [None] * world, [None] * world

    def run(rank):
        try:
            ctx = hps.Context(0)
            ctx.attach_local(grp, rank)
            el = hps.build_elements(ctx, prob)
            sk = hps.assemble_skeleton(el, prob)
            h = hps.build_hierarchy(sk)
            pc = hps.build_preconditioner(h, coarse_iters=4)
            res = {"rhs": sk.rhs(), "Mx": sk.apply(x), "Pv": pc.apply(v)}
            res["x"], res["rep"] = hps.fgmres(sk, sk.rhs(), pc, restart=prob.restart, tol=prob.tol)
            pe = hps.build_preconditioner(h, exact_coarse=True)
            res["Pe"] = pe.apply(v)
            res["direct"] = h.direct_solve(sk.rhs())
            res["field"] = sk.recover(res["x"])
            res["rank_world"] = ctx.rank_world
            out[rank] = res
        except Exception as exc:  # noqa: BLE001
            errs[rank] = exc

    threads = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in threads), "sharded run hung"
    failed = [(r, repr(e)) for r, e in enumerate(errs) if e is not None]
    assert not failed, failed
    return out


def test_nccl_attach_single_rank():
    # The NCCL communicator itself (init, one-rank world) on the real device;
    # multi-rank NCCL needs one GPU per rank and runs under bench.py --gpus N.
    import paper_2511_00735_b200 as hps
    prob = hps.problem(2, 0)
    ctx = hps.Context(0)
    ctx.attach_nccl(hps.nccl_unique_id(), 0, 1)
    assert ctx.rank_world == (0, 1)
    el = hps.build_elements(ctx, prob)
    sk = hps.assemble_skeleton(el, prob)
    pc = hps.build_preconditioner(hps.build_hierarchy(sk), coarse_iters=4)
    _, rep = hps.fgmres(sk, sk.rhs(), pc, restart=prob.restart, tol=prob.tol)
    assert rep["converged"]


@pytest.mark.parametrize("config,world", [(1, 2), (1, 4), (0, 2), (1, 8)])
def test_sharded_matches_single_gpu(config, world):
    import paper_2511_00735_b200 as hps
    prob = hps.problem(2, config)
    rng = np.random.default_rng(3)
    dim = 2 * (2 * prob.n * (prob.n - 1)) * (prob.order - 1)
    x = rng.standard_normal(dim) + 1j * rng.standard_normal(dim)
    v = rng.standard_normal(dim) + 1j * rng.standard_normal(dim)
    ref = _single(hps, prob, x, v)
    shards = _sharded(hps, prob, world, x, v)
    for rank, s in enumerate(shards):
        assert s["rank_world"] == (rank, world)
        assert relf(s["rhs"], ref["rhs"]) < 1e-12
        assert relf(s["Mx"], ref["Mx"]) < 1e-12
        assert relf(s["Pv"], ref["Pv"]) < 1e-10
        assert s["rep"]["converged"]
        assert abs(s["rep"]["iterations"] - ref["rep"]["iterations"]) <= 1
        assert relf(s["x"], ref["x"]) < 1e-9
        assert relf(s["Pe"], ref["Pe"]) < 1e-10          # exact coarse (dense inverse)
        assert relf(s["direct"], ref["direct"]) < 1e-9   # direct_solve
        assert relf(s["field"], ref["field"]) < 1e-9     # recover_solution
    # every rank holds the same replicated solution
    for s in shards[1:]:
        assert relf(s["x"], shards[0]["x"]) < 1e-12


def test_guard_trip_on_one_rank_rebuilds_on_all(monkeypatch):
    """The diagonal-pivot guard trips on rank 1 only: the ranks agree on it
    (allreduce) and all rebuild with partial pivoting together -- no
    mismatched collectives, same results as the single GPU."""
    import paper_2511_00735_b200 as hps
    prob = hps.problem(2, 1)
    rng = np.random.default_rng(4)
    dim = 2 * (2 * prob.n * (prob.n - 1)) * (prob.order - 1)
    x = rng.standard_normal(dim) + 1j * rng.standard_normal(dim)
    v = rng.standard_normal(dim) + 1j * rng.standard_normal(dim)
    ref = _single(hps, prob, x, v)
    monkeypatch.setenv("HPSB_TEST_GUARD_TRIP_RANK", "1")
    shards = _sharded(hps, prob, 4, x, v)
    for s in shards:
        assert relf(s["Pv"], ref["Pv"]) < 1e-10
        assert abs(s["rep"]["iterations"] - ref["rep"]["iterations"]) <= 1
        assert relf(s["x"], ref["x"]) < 1e-9


def _run_ranks(world, fn):
    grp_out, errs = [None] * world, [None] * world

    def run(rank):
        try:
            grp_out[rank] = fn(rank)
        except Exception as exc:  # noqa: BLE001
            errs[rank] = exc

    threads = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in threads), "sharded run hung"
    failed = [(r, repr(e)) for r, e in enumerate(errs) if e is not None]
    assert not failed, failed
    return grp_out


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_multi_rhs(world):
    """cfg4's setting (plane-wave right-hand sides, s = 0) on a 16 x 16 mesh at
    cfg4's kappa h (kappa = 600 * 16 / 256): the lockstep multi-RHS FGMRES on
    distributed vectors (owner-computes top merges, batched global-row and
    coefficient allreduces) matches the single GPU."""
    import paper_2511_00735_b200 as hps
    prob = hps.problem(2, 4, n=16, kappa=37.5)
    R = 4
    ctx = hps.Context(0)
    el = hps.build_elements(ctx, prob)
    sk = hps.assemble_skeleton(el, prob)
    pc = hps.build_preconditioner(hps.build_hierarchy(sk, factor_coarse=False), coarse_iters=4)
    rhs = np.stack([sk.rhs(b) for b in range(R)])
    X0, reps0 = hps.fgmres_batch(sk, rhs, pc, restart=60, tol=1e-8)
    assert all(r["converged"] for r in reps0)
    grp = hps.LocalGroup(world)

    def rank_run(rank):
        c = hps.Context(0)
        c.attach_local(grp, rank)
        e = hps.build_elements(c, prob)
        s = hps.assemble_skeleton(e, prob)
        p = hps.build_preconditioner(hps.build_hierarchy(s, factor_coarse=False), coarse_iters=4)
        r = np.stack([s.rhs(b) for b in range(R)])
        return hps.fgmres_batch(s, r, p, restart=60, tol=1e-8)

    for X, reps in _run_ranks(world, rank_run):
        for b in range(R):
            assert reps[b]["converged"]
            assert abs(reps[b]["iterations"] - reps0[b]["iterations"]) <= 1
            assert relf(X[b], X0[b]) < 1e-7


@pytest.mark.parametrize("world", [2, 8])
def test_sharded_krylov_variants(world):
    """Distributed vectors under single-pass MGS and the right-preconditioned
    gmres: every rank matches the single GPU."""
    import paper_2511_00735_b200 as hps
    prob = hps.problem(2, 1)
    ctx = hps.Context(0)
    el = hps.build_elements(ctx, prob)
    sk = hps.assemble_skeleton(el, prob)
    pc = hps.build_preconditioner(hps.build_hierarchy(sk, factor_coarse=False), coarse_iters=4)
    xm, rm = hps.fgmres(sk, sk.rhs(), pc, restart=50, tol=1e-10, reorthogonalize=False)
    xr, rr = hps.gmres(sk, sk.rhs(), restart=50, tol=1e-10, right_precond=pc)
    grp = hps.LocalGroup(world)

    def rank_run(rank):
        c = hps.Context(0)
        c.attach_local(grp, rank)
        e = hps.build_elements(c, prob)
        s = hps.assemble_skeleton(e, prob)
        p = hps.build_preconditioner(hps.build_hierarchy(s, factor_coarse=False), coarse_iters=4)
        a = hps.fgmres(s, s.rhs(), p, restart=50, tol=1e-10, reorthogonalize=False,
                       record_history=True)
        b = hps.gmres(s, s.rhs(), restart=50, tol=1e-10, right_precond=p)
        return a, b

    for (x1, r1), (x2, r2) in _run_ranks(world, rank_run):
        assert abs(r1["iterations"] - rm["iterations"]) <= 1 and relf(x1, xm) < 1e-9
        assert r1["basis_orthogonality"] < 1e-5  # single MGS pass (oracle: ~1e-6 on cfg1)
        assert abs(r2["iterations"] - rr["iterations"]) <= 1 and relf(x2, xr) < 1e-9


@pytest.mark.parametrize("world,gamma", [(2, 2), (4, 2), (4, 3)])
def test_sharded_gamma_cycle(world, gamma):
    """gamma-cycles (multigrid.cpp:66-80) on distributed vectors: the level
    residuals rc - M_{l+1} z sum the ranks' box rows on the global rows, the
    global levels run owner-computes; MG(v) and the FGMRES solve match the
    single GPU."""
    import paper_2511_00735_b200 as hps
    prob = hps.problem(2, 1)
    rng = np.random.default_rng(7)
    dim = 2 * (2 * prob.n * (prob.n - 1)) * (prob.order - 1)
    v = rng.standard_normal(dim) + 1j * rng.standard_normal(dim)
    ctx = hps.Context(0)
    el = hps.build_elements(ctx, prob)
    sk = hps.assemble_skeleton(el, prob)
    pc = hps.build_preconditioner(hps.build_hierarchy(sk, factor_coarse=False), gamma=gamma, coarse_iters=2)
    z0 = pc.apply(v)
    x0, r0 = hps.fgmres(sk, sk.rhs(), pc, restart=50, tol=1e-10)
    assert r0["converged"]
    grp = hps.LocalGroup(world)

    def rank_run(rank):
        c = hps.Context(0)
        c.attach_local(grp, rank)
        e = hps.build_elements(c, prob)
        s = hps.assemble_skeleton(e, prob)
        p = hps.build_preconditioner(hps.build_hierarchy(s, factor_coarse=False), gamma=gamma, coarse_iters=2)
        return p.apply(v), hps.fgmres(s, s.rhs(), p, restart=50, tol=1e-10)

    for z, (x, r) in _run_ranks(world, rank_run):
        assert relf(z, z0) < 1e-10
        assert r["converged"] and abs(r["iterations"] - r0["iterations"]) <= 1
        assert relf(x, x0) < 1e-9
