#!/bin/bash
# A/B of sed-made source variants on the cfg4 16-RHS apply (per-level profile) -- edit the variant lines per experiment.
cd "$GRAFT_REPO_ROOT"
b() { HPSB_PROFILE_LEVELS=1 timeout 600 python tools/vcycle_levels_batch.py 4 16 3 2>&1 | grep "per batched apply" | sed "s/^/$1 /"; }
variant() {  # $1 name, $2 file, $3 sed
  rm -rf /tmp/vb && cp -r "$GRAFT_REPO_ROOT" /tmp/vb && cd /tmp/vb/paper_2511_00735_b200 && \
    sed -i "$3" csrc/$2 && make -s -j 2>&1 | grep -i " error"; cd /tmp/vb; b $1; cd "$GRAFT_REPO_ROOT"
}
b base
variant stages2 zgemv_batch.cu 's/constexpr int BM = 64, BK = 16, STAGES = 3, THREADS = 256;/constexpr int BM = 64, BK = 16, STAGES = 2, THREADS = 256;/'
variant stages4 zgemv_batch.cu 's/constexpr int BM = 64, BK = 16, STAGES = 3, THREADS = 256;/constexpr int BM = 64, BK = 16, STAGES = 4, THREADS = 256;/'
