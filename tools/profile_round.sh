#!/bin/sh
# One GPU call that refreshes the round's evidence (run under gpurun):
#   the bench line (with the five configs), the bench's launch list, ncu
#   --set full captures of the pulse kernel (NS update), of the fused
#   tcgen05 forward (default IO, one pass) and of the bench's forward with
#   bound management (the in-kernel re-issue loop), and of drift_to on the
#   cfg5 tile.
#   Every ncu pass runs only after the same command exited 0 without ncu.
#   Output: gpurun_out/prof/
set -e
cd "$(dirname "$0")/.."
OUT=gpurun_out/prof
mkdir -p $OUT
python bench.py > $OUT/bench.json 2> $OUT/bench.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-configs > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_bench_steps2.csv python bench.py --steps 2 --warmup 1 \
    --no-cpu-baseline --no-configs > $OUT/ncu_launches.log 2>&1
python tools/profile_pulse.py --precision 1 --iters 2 > /dev/null
ncu --set full --import-source on --clock-control none -k regex:pulse_kernel -s 1 -c 1 -f \
    -o $OUT/pulse python tools/profile_pulse.py --precision 1 --iters 2 > $OUT/ncu_pulse.log 2>&1
python tools/time_mvm.py --iters 3 > /dev/null
ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 2 -c 1 -f \
    -o $OUT/tc_fwd python tools/time_mvm.py --iters 3 > $OUT/ncu_tc.log 2>&1
python tools/time_fwd_bench.py --only bm --iters 3 > /dev/null
ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 2 -c 1 -f \
    -o $OUT/tc_fwd_bm python tools/time_fwd_bench.py --only bm --iters 3 > $OUT/ncu_tc_bm.log 2>&1
python tools/time_drift.py --iters 2 > /dev/null
ncu --set full --import-source on --clock-control none -k regex:drift_kernel -s 1 -c 1 -f \
    -o $OUT/drift python tools/time_drift.py --iters 2 > $OUT/ncu_drift.log 2>&1
for r in pulse tc_fwd tc_fwd_bm drift; do
    python tools/ncu_summary.py $OUT/$r.ncu-rep --blocks > $OUT/$r.txt 2>&1 || true
done
