#!/usr/bin/env bash
# Shorter round evidence (after round_profile.sh): GPU tests, smoke, bench,
# the host drop-in breakdown, the ncu launch list of one solve and full
# captures of the SpMV and fused kernels. Usage: bash scripts/quick_round.sh <tag>
set -u
TAG=${1:-rq}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$OUT/gpu.txt" 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > "$OUT/pytest_gpu.txt" 2>&1
tail -2 "$OUT/pytest_gpu.txt"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.txt" 2>&1; tail -1 "$OUT/smoke.txt"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; tail -c 400 "$OUT/bench.json"; echo
timeout 300 python scripts/e2e_probe.py > "$OUT/e2e_probe.txt" 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file "$OUT/ncu_launches.csv" python scripts/one_solve.py poisson128 frsz2-32 > /dev/null 2>&1
python scripts/traffic_from_launches.py "$OUT/ncu_launches.csv" "$OUT/traffic.json" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:uslot_spmv -s 30 -c 1 -o "$OUT/ncu_spmv" \
    python scripts/one_solve.py poisson128 frsz2-32 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:arnoldi_fused -s 63 -c 1 -o "$OUT/ncu_fused" \
    python scripts/one_solve.py poisson128 frsz2-32 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:compress4 -s 2 -c 1 -o "$OUT/ncu_compress21" \
    python scripts/codec_one.py 21 > /dev/null 2>&1
ls "$OUT"
