for cfg in "8 8 2" "12 5 2" "10 6 2"; do
  set -- $cfg
  export CBGX_NVFLAGS_EXTRA="-DFUSED_WARPS=$1 -DFUSED_STEPS=$2 -DFUSED_CTAS_PER_SM=$3"
  python -c "from paper_2409_15468_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== warps=$1 steps=$2 ctas=$3"
  timeout 300 python -m pytest tests/test_solver_gpu.py -q -x --timeout 200 -k "tree_order or fused or bit_identical" 2>&1 | tail -1
  python bench.py --no-fp64 --no-e2e --no-codec --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_solve_phase_timed'], d['phase_ms_per_solve'])"
done
