"""Unpreconditioned GMRES (matvec + CGS2 only) repeated: iteration counts and
the bitwise spread of the solutions (determinism probe of the Krylov kernels).
usage: python tools/orth_probe.py CONFIG REPEATS ITERS"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_00735_b200 as hps  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
its = int(sys.argv[3]) if len(sys.argv) > 3 else 30
prob = hps.problem(2, cfg)
ctx = hps.Context(0)
el = hps.build_elements(ctx, prob)
sk = hps.assemble_skeleton(el, prob)
rhs = sk.rhs()
ys = [sk.apply(rhs) for _ in range(reps)]
print("matvec spread:", max(np.abs(y - ys[0]).max() for y in ys))
xs = []
for r in range(reps):
    x, rep = hps.fgmres(sk, rhs, None, restart=100, tol=1e-30, max_iters=its)
    xs.append(x)
print("gmres spread:", max(np.abs(x - xs[0]).max() for x in xs) / np.abs(xs[0]).max())
