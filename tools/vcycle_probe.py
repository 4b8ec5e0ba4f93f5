"""One preconditioner apply of a config (for ncu captures of the V-cycle kernels).
Usage: python tools/vcycle_probe.py [config] [applies]"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2511_00735_b200 as hps  # noqa: E402

cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
prob = hps.problem(2, cfgno, seed=cfgno)
ctx = hps.Context(0)
el = hps.build_elements(ctx, prob)
sk = hps.assemble_skeleton(el, prob)
hier = hps.build_hierarchy(sk, factor_coarse=False)
pc = hps.build_preconditioner(hier, coarse_iters=4)
v = torch.randn(2 * sk.dim, dtype=torch.float64, device="cuda")
z = torch.empty_like(v)
ctx.synchronize()
for _ in range(reps):
    hps._check(hps._lib.hpsb_precond_apply_dev(pc._h, ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(z.data_ptr())))
ctx.synchronize()
print("ok")
