import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2511_00735_b200 as hps
ctx = hps.Context(0)
for (n, N) in [(4, 4), (8, 4), (16, 4), (4, 8), (4, 16), (8, 8)]:
    p = hps.problem(0, 0, n=n, order=N, kappa=6.0)
    el = hps.build_elements(ctx, p); sk = hps.assemble_skeleton(el, p)
    h = hps.build_hierarchy(sk, factor_coarse=False)
    for depth in sorted({2, h.depth}):
        hh = hps.build_hierarchy(sk, depth=depth, factor_coarse=False)
        pc = hps.build_preconditioner(hh, coarse_iters=4, exact_coarse=True)
        R = 1
        rng = np.random.default_rng(1)
        X = rng.standard_normal((R, sk.dim)) + 1j * rng.standard_normal((R, sk.dim))
        xd = torch.from_numpy(X.view(np.float64)).cuda()
        zd = torch.zeros_like(xd)
        hps._check(hps._lib.hpsb_precond_apply_batch_dev(pc._h, xd.data_ptr(), zd.data_ptr(), R))
        ctx.synchronize()
        Z = zd.cpu().numpy().view(np.complex128).reshape(R, -1)
        ref = np.stack([pc.apply(X[b]) for b in range(R)])
        err = np.abs(Z - ref).max(axis=0)
        bad = np.nonzero(err > 1e-8 * np.abs(ref).max())[0]
        print(n, N, "depth", depth, "of", h.depth, "dim", sk.dim, "bad", len(bad), "first", bad[:4], "last", bad[-4:], flush=True)
