import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2511_00735_b200 as hps
ctx = hps.Context(0)
for spec in [dict(kind=0, config=0, n=4, order=4, kappa=6.0), dict(kind=2, config=2, n=8)]:
    p = hps.problem(**spec)
    el = hps.build_elements(ctx, p); sk = hps.assemble_skeleton(el, p)
    h = hps.build_hierarchy(sk, factor_coarse=False)
    for exact in (False, True):
        pc = hps.build_preconditioner(h, coarse_iters=4, exact_coarse=exact)
        for R in (1, 2):
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
            print(spec.get("n"), "exact", exact, "R", R, "max err", err.max(), "bad", len(bad), "of", sk.dim,
                  "first bad", bad[:8], flush=True)
