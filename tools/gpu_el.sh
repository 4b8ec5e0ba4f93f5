#!/bin/bash
# Element stage A/B: parity tests, then the cfg3 element probe for the tree and for sed-made variants.
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -q -p no:cacheprovider -k "element or iti or golden" 2>&1 | tail -3
b() { timeout 300 python tools/element_probe.py 3 4 prof 2>&1 | tail -1 | python -c "
import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('$1 element_iti ms/build', round(d['element_iti']['ms']/4,2))"; }
b base
variant() {  # $1 name, $2 file, $3 sed
  rm -rf /tmp/vb && cp -r "$GRAFT_REPO_ROOT" /tmp/vb && cd /tmp/vb/paper_2511_00735_b200 && \
    sed -i "$3" csrc/$2 && make -s -j 2>&1 | grep -i " error"; cd /tmp/vb; b $1; cd "$GRAFT_REPO_ROOT"
}
variant diag5 element_v5.cu 's/__launch_bounds__(V5DT, 6) v5_diag_kernel/__launch_bounds__(V5DT, 5) v5_diag_kernel/'
variant diag4 element_v5.cu 's/__launch_bounds__(V5DT, 6) v5_diag_kernel/__launch_bounds__(V5DT, 4) v5_diag_kernel/'
