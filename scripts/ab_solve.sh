#!/usr/bin/env bash
# A/B build variants on the bench solve (config 2, FRSZ2-32) and a short
# config-2 sweep of the other formats.
# Usage: bash scripts/ab_solve.sh "<nvcc flags A>" "<nvcc flags B>" ...
for flags in "$@"; do
  export CBGX_NVFLAGS_EXTRA="$flags"
  python -c "from paper_2409_15468_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== [$flags]"
  timeout 300 python -m pytest tests/test_solver_gpu.py -q -x --timeout 200 2>&1 | tail -1
  for i in 1 2; do
  timeout 300 python bench.py --no-fp64 --no-e2e --no-codec --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('  solve', d['value'], d['ms_per_solve_phase_timed'], d['phase_ms_per_solve'])"
  done
  timeout 600 python scripts/config_sweep.py --configs 2 --reps 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('  c2', d['format'], d['iterations'], d['ms_per_solve'])"
done
