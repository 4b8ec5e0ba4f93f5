#!/bin/bash
# Element stage: parity tests, then the cfg3 / cfg4 / cfg2 element probes (device time per build).
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -q -p no:cacheprovider -k "element or iti or golden" 2>&1 | tail -2
for c in 3 4 2; do timeout 300 python tools/element_probe.py $c 4 prof 2>&1 | tail -1 | python -c "
import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('cfg$c element_iti ms/build', round(d['element_iti']['ms']/4,2))"; done
