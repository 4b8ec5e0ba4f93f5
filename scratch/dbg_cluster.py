import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2511_00735_b200 as hps
from oracle import pyoracle as oracle
ctx = hps.Context(0)
for name, spec in [("cfg3_n4", dict(kind=2, config=3, n=4)), ("cfg2_n8", dict(kind=2, config=2, n=8)), ("cfg1", dict(kind=2, config=1))]:
    p = hps.problem(**spec)
    S = oracle.Session(p.n, p.order, p.kappa, p.eta, p.coeff, p.source, p.tside[0])
    el = hps.build_elements(ctx, p); sk = hps.assemble_skeleton(el, p)
    h = hps.build_hierarchy(sk, factor_coarse=False)
    pc = hps.build_preconditioner(h, coarse_iters=4)
    S.build_hierarchy(0, False); S.precond(depth=h.depth, gamma=1, coarse_iters=4)
    rng = np.random.default_rng(0)
    worst = 0; nd = 0
    for k in range(20):
        v = rng.standard_normal(sk.dim) + 1j * rng.standard_normal(sk.dim)
        a = pc.apply(v); b = pc.apply(v)
        nd += int(not np.array_equal(a, b))
        o = S.precond_apply(v)
        worst = max(worst, np.linalg.norm(a - o) / np.linalg.norm(o))
    x, rep = hps.fgmres(sk, sk.rhs(), pc, restart=100, tol=1e-10)
    xo, repo = S.solve(S.rhs(), True, restart=100, tol=1e-10)
    print(name, "precond worst", worst, "nondet", nd, "its", rep["iterations"], repo["iterations"], flush=True)
