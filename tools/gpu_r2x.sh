#!/bin/bash
# Round-2 GPU call X: determinism probe (stream orth vs legacy orth; cfg2 and cfg3).
cd "$GRAFT_REPO_ROOT"
for c in 2 3; do
  echo "== stream orth cfg$c"; timeout 600 python tools/determinism_probe.py $c 4 2>&1 | grep -v "Exception\|Traceback\|File \|AttributeError"
  echo "== legacy orth cfg$c"; HPSB_ORTH_LEGACY=1 timeout 600 python tools/determinism_probe.py $c 4 2>&1 | grep -v "Exception\|Traceback\|File \|AttributeError"
done
