#!/bin/sh
# One GPU call that refreshes the round's evidence (run under gpurun):
#   bench line, per-config lines, bench launch list, ncu --set full captures of
#   the pulse kernel and the tcgen05 contractions (TF32 fwd/bwd, 3xTF32 fwd).
# Every ncu pass runs only after the same command exited 0 without ncu.
set -e
cd "$(dirname "$0")/.."
OUT=gpurun_out/prof
mkdir -p $OUT
python bench.py > $OUT/bench.json 2> $OUT/bench.err
python tools/bench_configs.py > $OUT/configs.jsonl 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_bench_steps2.csv python bench.py --steps 2 --warmup 1 \
    --no-cpu-baseline > $OUT/ncu_launches.log 2>&1
python tools/profile_pulse.py --precision 1 --iters 2 --backward > /dev/null
ncu --set full --import-source on --clock-control none -k regex:pulse_kernel -s 1 -c 1 -f \
    -o $OUT/pulse python tools/profile_pulse.py --precision 1 --iters 2 > $OUT/ncu_pulse.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 2 -c 1 -f \
    -o $OUT/tc_tf32 python tools/profile_pulse.py --precision 1 --iters 2 --backward \
    > $OUT/ncu_tc.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:tc_gemm_kernel<.bool.1" -s 1 -c 1 -f -o $OUT/tc_tf32_bwd \
    python tools/profile_pulse.py --precision 1 --iters 2 --backward > $OUT/ncu_tcb.log 2>&1
python tools/profile_pulse.py --precision 2 --iters 2 > /dev/null
ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 1 -c 1 -f \
    -o $OUT/tc_x3 python tools/profile_pulse.py --precision 2 --iters 2 > $OUT/ncu_tcx3.log 2>&1
