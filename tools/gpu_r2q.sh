#!/bin/bash
# Round-2 GPU call Q: compute-sanitizer (memcheck / racecheck / synccheck) on
# the smoke path (cfg0) and a cfg1 preconditioned solve; cfg4 and cfg2 bench.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
cat > /tmp/san_cfg1.py <<'PY'
import sys; sys.path.insert(0, ".")
import paper_2511_00735_b200 as hps
prob = hps.problem(2, 1)
ctx = hps.Context(0)
el = hps.build_elements(ctx, prob); sk = hps.assemble_skeleton(el, prob)
h = hps.build_hierarchy(sk); pc = hps.build_preconditioner(h, coarse_iters=4)
x, rep = hps.fgmres(sk, sk.rhs(), pc, restart=prob.restart, tol=prob.tol)
print("cfg1 iterations", rep["iterations"], "converged", rep["converged"])
PY
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" \
      > gpurun_out/san_${tool}_cfg0.log 2>&1
  echo "$tool cfg0 rc=$?" >> gpurun_out/san_${tool}_cfg0.log
  timeout 1800 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san_cfg1.py \
      > gpurun_out/san_${tool}_cfg1.log 2>&1
  echo "$tool cfg1 rc=$?" >> gpurun_out/san_${tool}_cfg1.log
  tail -n 3 gpurun_out/san_${tool}_cfg0.log gpurun_out/san_${tool}_cfg1.log
done
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/bench_cfg4_q.json 2> gpurun_out/bench_cfg4_q.err
timeout 900 python bench.py --config 2 --steps 5 --warmup 3 > gpurun_out/bench_cfg2_q.json 2> gpurun_out/bench_cfg2_q.err
for c in 4 2; do python -c "
import json; d=json.load(open('gpurun_out/bench_cfg${c}_q.json'))
print({k: d.get(k) for k in ['value','setup','solve_ms_per_step','roofline_setup','roofline_gmres','iterations']})"; done
