#!/bin/bash
# Round-2 GPU call AQ: element update/trsm/back kernels -- 3-stage x 3 CTAs/SM vs 2-stage x 4 CTAs/SM (variant build).
cd "$GRAFT_REPO_ROOT"
b() { timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['setup'], d['kernels']['element_iti'])"; }
b A
rm -rf /tmp/vb && cp -r "$GRAFT_REPO_ROOT" /tmp/vb && cd /tmp/vb/paper_2511_00735_b200 && \
  sed -i "s/__launch_bounds__(V5T, 4)/__launch_bounds__(V5T, 5)/g" csrc/element_v5.cu && \
  grep -c "V5T, 5" csrc/element_v5.cu && make -s -j 2>&1 | grep -i " error"; cd /tmp/vb
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k element 2>&1 | tail -1
b B
