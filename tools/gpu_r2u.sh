#!/bin/bash
# Round-2 GPU call U: A/B of the persistent coarse GMRES grid (cfg3 bench solve time).
cd "$GRAFT_REPO_ROOT"
b() { timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['solve_ms_per_step'], d['roofline_gmres']['frac'])"; }
b "A coarse_wide"
rm -rf /tmp/vb && cp -r "$GRAFT_REPO_ROOT" /tmp/vb && cd /tmp/vb/paper_2511_00735_b200 && \
  sed -i 's/if (!cfg.exact_coarse \&\& !p->coarse_fused \&\& !p->coarse_cluster \&\& ci >= 1/if (false \&\& !cfg.exact_coarse \&\& !p->coarse_fused \&\& !p->coarse_cluster \&\& ci >= 1/' csrc/precond.cu && \
  grep -c "if (false && !cfg.exact_coarse" csrc/precond.cu && make -s -j 2>&1 | grep -i error; cd /tmp/vb
b "B split coarse"
