import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2511_00735_b200 as hps
ctx = hps.Context(0)
for (n, N) in [(4, 8), (4, 20), (8, 20)]:
    p = hps.problem(0, 0, n=n, order=N, kappa=6.0)
    el = hps.build_elements(ctx, p); sk = hps.assemble_skeleton(el, p)
    for R in (1, 3):
        rng = np.random.default_rng(1)
        X = rng.standard_normal((R, sk.dim)) + 1j * rng.standard_normal((R, sk.dim))
        xd = torch.from_numpy(X.view(np.float64)).cuda()
        yd = torch.zeros_like(xd)
        hps._check(hps._lib.hpsb_skeleton_apply_batch_dev(sk._h, xd.data_ptr(), yd.data_ptr(), R))
        ctx.synchronize()
        Y = yd.cpu().numpy().view(np.complex128).reshape(R, -1)
        ref = np.stack([sk.apply(X[b]) for b in range(R)])
        print(n, N, R, "matvec err", np.abs(Y - ref).max(), flush=True)
