#!/bin/bash
# Round-2 GPU call T: A/B of wide levels for cfg3 levels 7-8 (< 148 merges) via a variant build in /tmp.
cd "$GRAFT_REPO_ROOT"
run() { echo "== $1"; HPSB_PROFILE_LEVELS=1 timeout 300 python tools/vcycle_levels.py 3 5 2>&1 | grep "apply\|_L7 \|_L8 \|L7 \|L8 "; }
run "A cluster L7-8"
rm -rf /tmp/vb && cp -r "$GRAFT_REPO_ROOT" /tmp/vb && cd /tmp/vb/paper_2511_00735_b200 && \
  sed -i 's/if (!ng || ng >= 64 || l > h->sk->el->part.last_local) return -1;/if (!ng || ng >= 148 || l > h->sk->el->part.last_local) return -1;/' csrc/precond.cu && \
  grep -c "ng >= 148" csrc/precond.cu && make -s -j 2>&1 | grep -i error; cd /tmp/vb
run "B wide L7-8"
