#!/bin/bash
# Round-2 GPU call AJ: per-launch merge-GEMM efficiency at cfg3 (useful flops from HPSB_TRACE, times from events).
cd "$GRAFT_REPO_ROOT"
cat > /tmp/gemm_eff.py <<'PY'
import sys, os, re
sys.path.insert(0, ".")
import paper_2511_00735_b200 as hps
prob = hps.problem(2, 3)
ctx = hps.Context(0)
el = hps.build_elements(ctx, prob); sk = hps.assemble_skeleton(el, prob)
h = hps.build_hierarchy(sk, factor_coarse=False); ctx.synchronize()
del h
ctx.profile_reset(); ctx.profile(True)
h = hps.build_hierarchy(sk, factor_coarse=False); ctx.synchronize(); ctx.profile(False)
e = ctx.profile_entries()["zgemm_dmma"]
print("zgemm total", e)
PY
HPSB_TRACE=1 timeout 600 python /tmp/gemm_eff.py 2> gpurun_out/gemm_trace.txt | tail -2
grep -c "\[gemm\]" gpurun_out/gemm_trace.txt
