#!/usr/bin/env bash
for flags in "$@"; do
  export CBGX_NVFLAGS_EXTRA="$flags"
  python -c "from paper_2409_15468_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== [$flags]"
  timeout 300 python -m pytest tests/test_codec_gpu.py -q -x --timeout 200 2>&1 | tail -1
  timeout 300 python bench.py --no-fp64 --no-e2e --no-cpu-baseline --steps 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('  codec', {k: (v['compress_gbs'], v['decompress_gbs']) for k, v in d['codec'].items() if k.startswith('l')})"
done
