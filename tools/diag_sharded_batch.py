"""Diagnostic: sharded multi-RHS operators vs the single GPU (emulated ranks)."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_00735_b200 as hps

def relf(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)

prob = hps.problem(2, 4, n=16)
R, world = 3, 2
rng = np.random.default_rng(1)

def ops(ctx):
    el = hps.build_elements(ctx, prob)
    sk = hps.assemble_skeleton(el, prob)
    h = hps.build_hierarchy(sk, factor_coarse=False)
    pc = hps.build_preconditioner(h, coarse_iters=4)
    X = rng_x.copy()
    xd = torch.from_numpy(X.view(np.float64)).cuda()
    yd = torch.empty_like(xd); zd = torch.empty_like(xd)
    hps._check(hps._lib.hpsb_skeleton_apply_batch_dev(sk._h, xd.data_ptr(), yd.data_ptr(), R))
    hps._check(hps._lib.hpsb_precond_apply_batch_dev(pc._h, xd.data_ptr(), zd.data_ptr(), R))
    ctx.synchronize()
    Y = yd.cpu().numpy().view(np.complex128).reshape(R, -1)
    Z = zd.cpu().numpy().view(np.complex128).reshape(R, -1)
    z1 = pc.apply(X[0]); y1 = sk.apply(X[0])
    rhs = np.stack([sk.rhs(b) for b in range(R)])
    Xs, reps = hps.fgmres_batch(sk, rhs, pc, restart=60, tol=1e-8, max_iters=60)
    x1, rep1 = hps.fgmres(sk, rhs[0], pc, restart=60, tol=1e-8)
    return Y, Z, z1, y1, Xs, [r["iterations"] for r in reps], [r["final_residual"] for r in reps], rep1

dim = 2 * (2 * prob.n * (prob.n - 1)) * (prob.order - 1)
rng_x = rng.standard_normal((R, dim)) + 1j * rng.standard_normal((R, dim))
ref = ops(hps.Context(0))
print("single: its", ref[5], "res", ref[6], "single-rhs its", ref[7]["iterations"], flush=True)
grp = hps.LocalGroup(world)
out = [None] * world
def run(r):
    try:
        c = hps.Context(0); c.attach_local(grp, r); out[r] = ops(c)
    except Exception as e:
        out[r] = e
ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
[t.start() for t in ts]; [t.join() for t in ts]
for r, o in enumerate(out):
    if isinstance(o, Exception):
        print("rank", r, "error", o); continue
    print(f"rank {r}: batch matvec {relf(o[0], ref[0]):.2e} batch precond {relf(o[1], ref[1]):.2e} "
          f"single precond {relf(o[2], ref[2]):.2e} single matvec {relf(o[3], ref[3]):.2e} "
          f"its {o[5]} res {o[6]} single-rhs its {o[7]['iterations']}", flush=True)
