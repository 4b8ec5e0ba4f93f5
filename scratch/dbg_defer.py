import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2511_00735_b200 as hps
ctx = hps.Context(0)
prob = hps.problem(1, 0, n=8, order=8, kappa=float(sys.argv[1]) if len(sys.argv) > 1 else 0.0)
def run(sync_after_el, sync_after_sk):
    el = hps.build_elements(ctx, prob)
    if sync_after_el: ctx.synchronize()
    sk = hps.assemble_skeleton(el, prob)
    if sync_after_sk: ctx.synchronize()
    rhs = sk.rhs()
    T, H = el.iti()
    hier = hps.build_hierarchy(sk, 2)
    pc = hps.build_preconditioner(hier, 2, 1, 4, False)
    g, r = hps.fgmres(sk, rhs, pc, 50, 1e-10, 500, 0)
    f = sk.recover(g)
    return rhs, T, g, f, r["iterations"]
base = run(True, True)
for a in [(False, False), (True, False), (False, True)]:
    o = run(*a)
    print(a, [float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)) for x, y in zip(o[:4], base[:4])], o[4], base[4])
