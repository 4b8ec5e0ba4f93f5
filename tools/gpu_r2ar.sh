#!/bin/bash
# Round-2 GPU call AR: tuning A/B of the TMA-ring kernels (variant builds; cfg3 bench solve time).
cd "$GRAFT_REPO_ROOT"
b() { timeout 900 python bench.py --steps 4 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('$1', round(d['solve_ms_per_step'],2), d['iterations'][0], {n: k[n]['ms'] for n in ('vcycle_up','vcycle_down','gmres_orth','skeleton_matvec') if n in k})"; }
b base
variant() {  # $1 name, $2 file, $3 sed
  rm -rf /tmp/vb && cp -r "$GRAFT_REPO_ROOT" /tmp/vb && cd /tmp/vb/paper_2511_00735_b200 && \
    sed -i "$3" csrc/$2 && make -s -j 2>&1 | grep -i " error"; cd /tmp/vb; b $1; cd "$GRAFT_REPO_ROOT"
}
variant ns2 vcycle_stream.cu 's/  const int ns = 3;/  const int ns = 2;/'
variant cta653 vcycle_stream.cu 's/const int ctas_per_sm = cw == 4 ? 5 : cw == 8 ? 4 : 2;/const int ctas_per_sm = cw == 4 ? 6 : cw == 8 ? 5 : 3;/'
