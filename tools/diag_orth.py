"""Diagnostic: Arnoldi basis orthogonality of the GPU FGMRES vs the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_00735_b200 as hps
from oracle import pyoracle
for cfg, depth in [(0, 0), (1, 3), (1, 0), (2, 0)]:
    p = hps.problem(2, cfg)
    ctx = hps.Context(0)
    el = hps.build_elements(ctx, p); sk = hps.assemble_skeleton(el, p)
    h = hps.build_hierarchy(sk, factor_coarse=False)
    pc = hps.build_preconditioner(h, depth=depth or h.depth, coarse_iters=4)
    S = pyoracle.Session(p.n, p.order, p.kappa, p.eta, p.coeff, p.source, p.tside[0])
    S.build_hierarchy(0, False); S.precond(depth=depth or h.depth, gamma=1, coarse_iters=4)
    for reorth in (True, False):
        x, rep = hps.fgmres(sk, sk.rhs(), pc, restart=p.restart, tol=p.tol, record_history=True,
                            reorthogonalize=reorth)
        xo, repo = S.solve(S.rhs(), True, restart=p.restart, tol=p.tol, reorth=reorth, record_history=True)
        print(f"cfg{cfg} depth {depth or h.depth} reorth {reorth}: gpu its {rep['iterations']} orth "
              f"{rep['basis_orthogonality']:.2e} | oracle its {repo['iterations']} orth "
              f"{repo['basis_orthogonality']:.2e}", flush=True)
    x, rep = hps.gmres(sk, sk.rhs(), restart=30, tol=1e-8, max_iters=30, record_history=True)
    xo, repo = S.solve(S.rhs(), False, restart=30, tol=1e-8, max_iters=30, reorth=True, record_history=True)
    print(f"  unprec 30 its: gpu orth {rep['basis_orthogonality']:.2e} oracle {repo['basis_orthogonality']:.2e}")
    pc.close(); h.close(); sk.close(); el.close(); ctx.close()
