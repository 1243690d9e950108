#!/usr/bin/env bash
# A/B build variants on the bench solve only (FRSZ2-32, config 2): solve ms
# and the per-phase split, twice per variant.
# Usage: bash scripts/ab_quick.sh "<nvcc flags A>" "<nvcc flags B>" ...
for flags in "$@"; do
  export CBGX_NVFLAGS_EXTRA="$flags"
  python -c "from paper_2409_15468_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== [$flags]"
  for i in 1 2; do
  timeout 300 python bench.py --no-fp64 --no-e2e --no-codec --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['phase_ms_per_solve']; print('  solve', d['value'], 'phased', d['ms_per_solve_phase_timed'], 'spmv', p['spmv'], 'ortho', p['ortho'])"
  done
done
