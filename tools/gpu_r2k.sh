#!/bin/bash
# Round-2 GPU call K: stream-level PDL / level-range experiment (cfg3 V-cycle).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
run() { echo "== $1"; HPSB_PROFILE_LEVELS=1 timeout 300 python tools/vcycle_levels.py 3 5 2>&1 | grep -v "Exception\|Traceback\|File\|AttributeError" | head -${2:-1}; }
run "A early trigger" 8
HPSB_NO_PDL=1 run "A no PDL"
HPSB_STREAM_MIN_ROWS=97 run "A min rows 97" 8
rm -rf /tmp/vb && cp -r "$GRAFT_REPO_ROOT" /tmp/vb && cd /tmp/vb/paper_2511_00735_b200 && \
  touch csrc/vcycle_stream.cu && make -s -j EXTRA_NVFLAGS=-DHPSB_STREAM_LATE_TRIGGER 2>&1 | grep -i error; cd /tmp/vb
run "B late trigger" 8
HPSB_STREAM_MIN_ROWS=97 run "B min rows 97" 8
