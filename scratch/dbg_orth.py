import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2511_00735_b200 as hps
ctx = hps.Context(0)
p = hps.problem(kind=2, config=3, n=4)
el = hps.build_elements(ctx, p); sk = hps.assemble_skeleton(el, p)
h = hps.build_hierarchy(sk, factor_coarse=False)
pc = hps.build_preconditioner(h, coarse_iters=4)
x, rep = hps.fgmres(sk, sk.rhs(), pc, restart=100, tol=1e-10)
print("its", rep["iterations"], file=sys.stderr)
