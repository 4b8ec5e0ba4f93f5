"""Latency probe for the small (L2-resident) configurations.

Separates host enqueue time from device time for the pieces of one FGMRES
iteration: the preconditioner apply, the interface matvec, and a whole solve.
Usage: python tools/latency_probe.py [config]
"""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_00735_b200 as hps  # noqa: E402


def main():
    cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    prob = hps.problem(2, cfgno, seed=1)
    ctx = hps.Context(0)
    el = hps.build_elements(ctx, prob)
    sk = hps.assemble_skeleton(el, prob)
    hier = hps.build_hierarchy(sk, factor_coarse=False)
    pc = hps.build_preconditioner(hier, coarse_iters=4)
    n = sk.dim
    v = torch.randn(2 * n, dtype=torch.float64, device="cuda")
    z = torch.empty_like(v)
    w = torch.empty_like(v)
    ctx.synchronize()
    lib = hps._lib
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731

    def timeit(label, fn, reps=200):
        for _ in range(10):
            fn()
        ctx.synchronize()
        l0 = ctx.launches
        t0 = time.perf_counter()
        ctx.timer_start()
        for _ in range(reps):
            fn()
        t1 = time.perf_counter()
        dev = ctx.timer_stop()
        t2 = time.perf_counter()
        print(f"{label:28s} device {1e6 * dev / reps:8.1f} us  host enqueue {1e6 * (t1 - t0) / reps:8.1f} us"
              f"  wall {1e6 * (t2 - t0) / reps:8.1f} us  launches {(ctx.launches - l0) / reps:.1f}")

    timeit("precond apply", lambda: hps._check(lib.hpsb_precond_apply_dev(pc._h, P(v), P(z))))
    timeit("skeleton apply", lambda: hps._check(lib.hpsb_skeleton_apply_dev(sk._h, P(z), P(w))))

    def both():
        hps._check(lib.hpsb_precond_apply_dev(pc._h, P(v), P(z)))
        hps._check(lib.hpsb_skeleton_apply_dev(sk._h, P(z), P(w)))

    timeit("precond + matvec", both)
    cfg = hps.KrylovConfig(prob.restart, prob.tol, 2000, 0, 1)
    x = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        rep = hps.SolveReport()
        t0 = time.perf_counter()
        hps._check(lib.hpsb_fgmres_dev(sk._h, pc._h, ctypes.c_void_p(sk.rhs_dev_ptr(0)), P(x), cfg,
                                       ctypes.byref(rep)), allow=(hps.OK,))
        t1 = time.perf_counter()
        print(f"fgmres: {rep.iterations} its, device {1e6 * rep.seconds / rep.iterations:.1f} us/it, "
              f"wall {1e6 * (t1 - t0) / rep.iterations:.1f} us/it")




def coarse_slope():
    """Preconditioner apply device time vs coarse_iters (the coarse solve's per-step cost)."""
    cfgno = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    prob = hps.problem(2, cfgno, seed=1)
    ctx = hps.Context(0)
    el = hps.build_elements(ctx, prob)
    sk = hps.assemble_skeleton(el, prob)
    hier = hps.build_hierarchy(sk, factor_coarse=False)
    n = sk.dim
    v = torch.randn(2 * n, dtype=torch.float64, device="cuda")
    z = torch.empty_like(v)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    for ci in (1, 2, 4, 8):
        pc = hps.build_preconditioner(hier, coarse_iters=ci)
        for _ in range(10):
            hps._check(hps._lib.hpsb_precond_apply_dev(pc._h, P(v), P(z)))
        ctx.synchronize()
        ctx.timer_start()
        for _ in range(200):
            hps._check(hps._lib.hpsb_precond_apply_dev(pc._h, P(v), P(z)))
        dev = ctx.timer_stop()
        print(f"coarse_iters={ci}: precond apply device {1e6 * dev / 200:.1f} us")
        del pc


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "coarse":
        coarse_slope()
    else:
        main()
