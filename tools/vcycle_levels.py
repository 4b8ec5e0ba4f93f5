"""Per-level view of the V-cycle (CUDA events per launch, HPSB_PROFILE_LEVELS
labels): ms, algorithmic bytes and GB/s per level label over `applies`
preconditioner applies.  Usage: HPSB_PROFILE_LEVELS=1 python tools/vcycle_levels.py [config] [applies]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_00735_b200 as hps  # noqa: E402

cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
prob = hps.problem(2, cfgno, seed=cfgno)
ctx = hps.Context(0)
el = hps.build_elements(ctx, prob)
sk = hps.assemble_skeleton(el, prob)
hier = hps.build_hierarchy(sk, factor_coarse=False)
pc = hps.build_preconditioner(hier, coarse_iters=4)
v = torch.randn(2 * sk.dim, dtype=torch.float64, device="cuda")
z = torch.empty_like(v)
ctx.synchronize()
ctx.timer_start()
for _ in range(reps):
    hps._check(hps._lib.hpsb_precond_apply_dev(pc._h, ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(z.data_ptr())))
t = ctx.timer_stop()
print(f"cfg{cfgno}: {1e3 * t / reps:.3f} ms per apply (PDL on), {pc.bytes_per_apply / 1e9:.3f} GB "
      f"-> {pc.bytes_per_apply * reps / t / 1e9:.0f} GB/s")
ctx.profile_reset()
ctx.profile(True)
for _ in range(reps):
    hps._check(hps._lib.hpsb_precond_apply_dev(pc._h, ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(z.data_ptr())))
ctx.synchronize()
ctx.profile(False)
tot = 0.0
for name, d in sorted(ctx.profile_entries().items(), key=lambda kv: -kv[1]["ms"]):
    tot += d["ms"]
    print(f"{name:32s} {d['launches'] // reps:5d} launches {d['ms'] / reps:8.3f} ms  "
          f"{d['bytes'] / reps / 1e6:9.1f} MB  {d['bytes'] / max(d['ms'], 1e-9) / 1e6:7.0f} GB/s")
print(f"sum (events, no PDL) {tot / reps:.3f} ms per apply")
