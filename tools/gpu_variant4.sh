#!/bin/bash
# A/B of sed-made source variants on the cfg4 16-RHS apply -- edit the variant lines per experiment.
cd "$GRAFT_REPO_ROOT"
b() { HPSB_PROFILE_LEVELS=1 timeout 600 python tools/vcycle_levels_batch.py 4 16 3 2>&1 | grep "per batched apply" | sed "s/^/$1 /"; }
variant() {  # $1 name, $2 file, $3 sed
  rm -rf /tmp/vb && cp -r "$GRAFT_REPO_ROOT" /tmp/vb && cd /tmp/vb/paper_2511_00735_b200 && \
    sed -i "$3" csrc/$2 && make -s -j 2>&1 | grep -i " error"; cd /tmp/vb; b $1; cd "$GRAFT_REPO_ROOT"
}
b base
variant i2 zgemv_batch.cu 's/static constexpr int WN = BN \/ 16, I = BN \/ 16; /static constexpr int WN = BN \/ 16, I = 2; /'
