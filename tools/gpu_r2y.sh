#!/bin/bash
# Round-2 GPU call Y: bisect the orth_stream non-determinism with variant builds.
cd "$GRAFT_REPO_ROOT"
variant() {  # $1 name, $2 extra nvcc flags
  rm -rf /tmp/vb && cp -r "$GRAFT_REPO_ROOT" /tmp/vb && cd /tmp/vb/paper_2511_00735_b200 && \
    touch csrc/krylov.cu && make -s -j EXTRA_NVFLAGS="$2" 2>&1 | grep -i " error"; cd /tmp/vb
  echo "== $1"; timeout 600 python tools/orth_probe.py 3 4 40 2>&1 | grep "spread"
  cd "$GRAFT_REPO_ROOT"
}
echo "== legacy"; HPSB_ORTH_LEGACY=1 timeout 600 python tools/orth_probe.py 3 4 40 2>&1 | grep "spread"
variant "base" ""
variant "proxy fence" "-DHPSB_OS_PROXY_FENCE"
variant "all warps" "-DHPSB_OS_ALLWARPS"
