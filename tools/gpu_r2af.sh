#!/bin/bash
# Round-2 GPU call AF: sharded gamma-cycle tests + gamma tests + sharded suite.
cd "$GRAFT_REPO_ROOT"
timeout 1500 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 900 -rf -k "sharded or gamma" 2>&1 | tail -8
