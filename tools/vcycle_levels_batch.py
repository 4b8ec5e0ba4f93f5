"""Per-level view of the multi-RHS V-cycle (CUDA events per launch,
HPSB_PROFILE_LEVELS labels) for R right-hand sides.
Usage: HPSB_PROFILE_LEVELS=1 python tools/vcycle_levels_batch.py [config] [R] [applies]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_00735_b200 as hps  # noqa: E402

cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 4
R = int(sys.argv[2]) if len(sys.argv) > 2 else 16
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
prob = hps.problem(2, cfgno, seed=cfgno)
ctx = hps.Context(0)
el = hps.build_elements(ctx, prob)
sk = hps.assemble_skeleton(el, prob)
hier = hps.build_hierarchy(sk, factor_coarse=False)
pc = hps.build_preconditioner(hier, coarse_iters=4)
v = torch.randn(2 * sk.dim * R, dtype=torch.float64, device="cuda")
z = torch.empty_like(v)
apply = lambda: hps._check(hps._lib.hpsb_precond_apply_batch_dev(pc._h, ctypes.c_void_p(v.data_ptr()),
                                                                 ctypes.c_void_p(z.data_ptr()), R))
apply()
ctx.synchronize()
ctx.timer_start()
for _ in range(reps):
    apply()
t = ctx.timer_stop()
print(f"cfg{cfgno} R={R}: {1e3 * t / reps:.3f} ms per batched apply")
ctx.profile_reset()
ctx.profile(True)
for _ in range(reps):
    apply()
ctx.synchronize()
ctx.profile(False)
tot = 0.0
for name, d in sorted(ctx.profile_entries().items(), key=lambda kv: -kv[1]["ms"]):
    tot += d["ms"]
    print(f"{name:34s} {d['launches'] // reps:5d} launches {d['ms'] / reps:8.3f} ms  "
          f"{d['flops'] / reps / 1e9:9.1f} GF  {d['flops'] / max(d['ms'], 1e-9) / 1e9:7.2f} TF/s")
print(f"sum (events) {tot / reps:.3f} ms per apply")
