#!/usr/bin/env bash
# A/B build variants: CGS micro (config 4) per format + read sweep + solve.
for flags in "$@"; do
  export CBGX_NVFLAGS_EXTRA="$flags"
  python -c "from paper_2409_15468_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== [$flags]"
  timeout 300 python -m pytest tests/test_cgs_gpu.py -q -x --timeout 200 2>&1 | tail -1
  timeout 300 python scripts/cgs_micro.py --k 20,100 --formats frsz2-32,frsz2-21,frsz2-16 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for f,v in d['results'].items(): print('  cgs', f, {k:(r['dot_frac'],r['update_frac']) for k,r in v.items()})"
  timeout 300 python scripts/read_bench.py --formats frsz2-32,frsz2-16 --intensities 1 --log2-elements 27 2>&1 | tail -2
  timeout 300 python bench.py --no-fp64 --no-e2e --no-codec --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('  solve', d['value'], d['phase_ms_per_solve'])"
done
