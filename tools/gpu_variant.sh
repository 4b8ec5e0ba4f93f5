#!/bin/bash
# A/B of sed-made source variants on the cfg3 bench; edit the variant lines per experiment.
cd "$GRAFT_REPO_ROOT"
b() { timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('$1', 'setup', round(d['setup']['ms_per_step'],2), 'solve', round(d['solve_ms_per_step'],2), d['iterations'][0], {n: k[n]['ms'] for n in ('zgemm_dmma','element_iti','vcycle_up','vcycle_down','coarse_wide','skeleton_matvec','gmres_orth') if n in k})"; }
variant() {  # $1 name, $2 file, $3 sed
  rm -rf /tmp/vb && cp -r "$GRAFT_REPO_ROOT" /tmp/vb && cd /tmp/vb/paper_2511_00735_b200 && \
    sed -i "$3" csrc/$2 && make -s -j 2>&1 | grep -i " error"; cd /tmp/vb; b $1; cd "$GRAFT_REPO_ROOT"
}
b base
variant slots6 vcycle_wide.cu 's/constexpr int kWideSlots = 4;/constexpr int kWideSlots = 6;/'
variant slots8 vcycle_wide.cu 's/constexpr int kWideSlots = 4;/constexpr int kWideSlots = 8;/'
variant slots3 vcycle_wide.cu 's/constexpr int kWideSlots = 4;/constexpr int kWideSlots = 3;/'
