#!/usr/bin/env bash
# Round evidence on one B200: tests, bench (both arms), config-4 CGS micro,
# SpMV micro, ncu launch list of one solve (with DRAM bytes per launch), and
# full ncu captures of the hot kernels.
# Usage (via gpurun): bash scripts/round_profile.sh <tag>
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$OUT/gpu.txt" 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > "$OUT/pytest_gpu.txt" 2>&1
tail -3 "$OUT/pytest_gpu.txt"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; tail -c 600 "$OUT/bench.json"; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_reference.json" 2>&1; tail -c 300 "$OUT/bench_reference.json"; echo
timeout 600 python scripts/cgs_micro.py --k 10,20,50,100,150,200 --formats frsz2-32,frsz2-21,frsz2-16,f32,f64 > "$OUT/cgs_micro.txt" 2>&1
timeout 300 python scripts/spmv_micro.py > "$OUT/spmv_micro.txt" 2>&1
# launch list of one solve (cold-cache, serialised: compare shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file "$OUT/ncu_launches.csv" python scripts/one_solve.py poisson128 frsz2-32 > /dev/null 2>&1
python scripts/traffic_from_launches.py "$OUT/ncu_launches.csv" "$OUT/traffic.json" > /dev/null 2>&1
# full captures: fused orthogonalisation (mid-cycle launch), dictionary SpMV, codec, CGS micro at n = 2^26
timeout 600 ncu --set full --clock-control none --import-source on -k regex:arnoldi_fused -s 63 -c 1 -o "$OUT/ncu_fused" \
    python scripts/one_solve.py poisson128 frsz2-32 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:uslot_spmv -s 30 -c 1 -o "$OUT/ncu_spmv" \
    python scripts/one_solve.py poisson128 frsz2-32 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decompress4 -s 3 -c 1 -o "$OUT/ncu_decompress" \
    python scripts/quick_perf.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:compress4 -s 3 -c 1 -o "$OUT/ncu_compress" \
    python scripts/quick_perf.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:compress4 -s 2 -c 1 -o "$OUT/ncu_compress21" \
    python scripts/codec_one.py 21 > /dev/null 2>&1
# split CGS kernels (dynamic tiles) at n = 2^26, k = 100, per FRSZ2 format: the
# reports stay on the box (size), their raw metric pages come back as CSV
for f in frsz2-32 frsz2-21 frsz2-16; do
  for kk in dot update; do
    timeout 300 ncu --set full --clock-control none --import-source on -k regex:cgs_${kk}_dyn -s 1 -c 1 -o /tmp/ncu_cgs_${kk}_$f \
        python scripts/cgs_micro.py --k 100 --formats $f --reps 2 > /dev/null 2>&1
    ncu -i /tmp/ncu_cgs_${kk}_$f.ncu-rep --page raw --csv > "$OUT/ncu_cgs_${kk}_${f}_raw.csv" 2>&1
  done
done
timeout 900 python scripts/read_bench.py > "$OUT/read_bench.csv" 2>&1
timeout 1800 python scripts/config_sweep.py --configs 2,3 > "$OUT/config_sweep_c2_c3.jsonl" 2>&1
timeout 1800 python scripts/config_sweep.py --configs 5 --reps 1 > "$OUT/config_sweep_c5.jsonl" 2>&1
ls -la "$OUT"
