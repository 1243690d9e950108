#!/usr/bin/env bash
# A/B build variants on the GPU box: each argument is one CBGX_NVFLAGS_EXTRA
# string; for each: rebuild, quick parity tests, spmv micro, solver bench.
for flags in "$@"; do
  export CBGX_NVFLAGS_EXTRA="$flags"
  python -c "from paper_2409_15468_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== [$flags]"
  timeout 300 python -m pytest tests/test_solver_gpu.py -q -x --timeout 200 -k "staged or tree_order or stencil" 2>&1 | tail -1
  timeout 300 python scripts/spmv_micro.py 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  spmv', d['kind'], d['nx'], d.get('staged_us'), d.get('staged_frac'))"
  timeout 300 python bench.py --no-fp64 --no-e2e --no-codec --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('  solve', d['value'], d['ms_per_solve_phase_timed'], d['phase_ms_per_solve'])"
done
