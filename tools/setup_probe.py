"""One cfg setup (elements -> skeleton -> hierarchy -> preconditioner) after a
warm-up build; used under ncu to list the setup launches of one build.
usage: python tools/setup_probe.py CONFIG [BUILDS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_00735_b200 as hps  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
builds = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prob = hps.problem(2, cfg)
ctx = hps.Context(0)
for b in range(builds):
    el = hps.build_elements(ctx, prob)
    sk = hps.assemble_skeleton(el, prob)
    hier = hps.build_hierarchy(sk, factor_coarse=False)
    pc = hps.build_preconditioner(hier, coarse_iters=4)
    ctx.synchronize()
    print(f"build {b}: hierarchy device {1e3 * hier.build_seconds:.1f} ms", flush=True)
    del pc, hier, sk, el
