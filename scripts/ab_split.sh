#!/usr/bin/env bash
# A/B build variants of the split CGS kernels: config-4 micro per format.
# Usage: bash scripts/ab_split.sh "<nvcc flags A>" "<nvcc flags B>" ...
for flags in "$@"; do
  export CBGX_NVFLAGS_EXTRA="$flags"
  python -c "from paper_2409_15468_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== [$flags]"
  timeout 300 python scripts/cgs_micro.py --k 20,100 --formats ${AB_FORMATS:-frsz2-32,frsz2-21,frsz2-16} 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for f,v in d['results'].items(): print('  cgs', f, {k:(r['dot_frac'],r['update_frac']) for k,r in v.items()})"
done
