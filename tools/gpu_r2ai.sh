#!/bin/bash
# Round-2 GPU call AI: stream levels with prefetched output bases -- determinism, parity subset, levels, bench.
cd "$GRAFT_REPO_ROOT"
timeout 600 python tools/determinism_probe.py 3 3 2>&1 | grep "iterations\|solution\|MG"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "precond or golden or gamma or sharded or level" 2>&1 | tail -2
HPSB_PROFILE_LEVELS=1 timeout 300 python tools/vcycle_levels.py 3 5 2>&1 | grep "apply\|stream"
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['solve_ms_per_step'], d['roofline_gmres']['frac'], d['iterations'])"
