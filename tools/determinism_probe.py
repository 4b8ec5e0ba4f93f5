"""Repeat a preconditioned FGMRES solve and report iteration counts and the
bitwise spread of the solutions (race / determinism probe).
usage: python tools/determinism_probe.py CONFIG REPEATS"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_00735_b200 as hps  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
prob = hps.problem(2, cfg)
ctx = hps.Context(0)
el = hps.build_elements(ctx, prob)
sk = hps.assemble_skeleton(el, prob)
h = hps.build_hierarchy(sk, factor_coarse=False)
pc = hps.build_preconditioner(h, coarse_iters=4)
rhs = sk.rhs()
xs, its = [], []
for r in range(reps):
    x, rep = hps.fgmres(sk, rhs, pc, restart=prob.restart, tol=prob.tol)
    xs.append(x)
    its.append(rep["iterations"])
v = rhs.copy()
zs = [pc.apply(v) for _ in range(reps)]
print(f"cfg{cfg} iterations {its}")
print("solution max |x_r - x_0| / |x_0|:", max(np.abs(x - xs[0]).max() for x in xs) / np.abs(xs[0]).max())
print("MG(v) max |z_r - z_0|:", max(np.abs(z - zs[0]).max() for z in zs))
