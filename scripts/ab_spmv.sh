#!/usr/bin/env bash
# A/B build variants on the SpMV micro-bench (scripts/spmv_micro.py).
for flags in "$@"; do
  export CBGX_NVFLAGS_EXTRA="$flags"
  python -c "from paper_2409_15468_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== [$flags]"
  timeout 300 python scripts/spmv_micro.py 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('  kind', d['kind'], d['nx'], 'staged', d.get('staged_us'), 'dict', d['dict_us'], 'x', d.get('dict_speedup'))"
done
