#!/bin/bash
# Round-2 GPU call P: A/B of the stream kernel on cfg3 level 1 (variant built in /tmp).
cd "$GRAFT_REPO_ROOT"
run() { echo "== $1"; HPSB_PROFILE_LEVELS=1 timeout 300 python tools/vcycle_levels.py 3 5 2>&1 | grep "apply\|L1 \|_L1"; }
run "A small L1"
rm -rf /tmp/vb && cp -r "$GRAFT_REPO_ROOT" /tmp/vb && cd /tmp/vb/paper_2511_00735_b200 && \
  sed -i 's/if (bytes < 96e3 \* std::max(ng, 1)) return -1;/if (bytes < 0) return -1;/' csrc/precond.cu && \
  make -s -j 2>&1 | grep -i error; cd /tmp/vb
run "B stream L1"
