import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2511_00735_b200 as hps
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ctx = hps.Context(0)
p = hps.problem(kind=2, config=cfg)
el = hps.build_elements(ctx, p); sk = hps.assemble_skeleton(el, p)
h = hps.build_hierarchy(sk, factor_coarse=False)
pc = hps.build_preconditioner(h, coarse_iters=4)
rng = np.random.default_rng(0)
v = rng.standard_normal(sk.dim) + 1j * rng.standard_normal(sk.dim)
a = pc.apply(v)
print("apply finite", np.isfinite(a).all(), np.linalg.norm(a), flush=True)
try:
    x, rep = hps.fgmres(sk, sk.rhs(), pc, restart=p.restart, tol=p.tol)
    print("fgmres", rep)
except hps.HpsError as e:
    print("HpsError", e.args)
