#!/usr/bin/env bash
# A/B build variants on the dictionary SpMV probe (scripts/pell_probe.py,
# every coding level) and the bench solve. Usage: ab_ppat.sh "<flags>" ...
for flags in "$@"; do
  export CBGX_NVFLAGS_EXTRA="$flags"
  python -c "from paper_2409_15468_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== [$flags]"
  timeout 200 python scripts/pell_probe.py 128 2>&1 | grep "layout=(4"
  timeout 200 python scripts/pell_probe.py 256 2 2>&1 | grep "layout=(4"
  timeout 300 python bench.py --steps 20 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('  bench', d['value'], 'spmv', d['phase_ms_per_solve']['spmv'], 'e2e', round(d['e2e']['value'], 3))"
done
