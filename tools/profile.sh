#!/bin/bash
# Profiling recipe (B200_PROFILING.md) for one round; run under gpurun from the repo root:
#   gpurun -- 'bash tools/profile.sh rNN'
# 1) plain bench line, 2) the ncu launch list of the bench command after it exits 0,
# 3) `ncu --set full` captures of the top kernels from tools/prof_driver.py (after the
#    same command exited 0 without ncu).
set -u
R=${1:-r01}
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_${R}.json 2> gpurun_out/bench_${R}.err
echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain_${R}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${R}.csv $CMD > gpurun_out/ncu_launch_${R}.log 2>&1
echo "launch list rc=$?"
python tools/prof_driver.py sweep > gpurun_out/plain_sweep_${R}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'sweep2d_reg_kernel|sweep2d_kernel' -s 50 -c 1 \
    -o gpurun_out/prof_sweep2d_${R} python tools/prof_driver.py sweep > gpurun_out/ncu_sweep2d_${R}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep1d_kernel -s 50 -c 1 \
    -o gpurun_out/prof_sweep1d_${R} python tools/prof_driver.py sweep > gpurun_out/ncu_sweep1d_${R}.log 2>&1
echo "sweep full rc=$?"
python tools/prof_driver.py layer > gpurun_out/plain_layer_${R}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'gemm_kernel|input_kernel|output_kernel' -s 3 -c 3 \
    -o gpurun_out/prof_layer_${R} python tools/prof_driver.py layer > gpurun_out/ncu_layer_${R}.log 2>&1
echo "layer full rc=$?"
python tools/tf32_time.py > gpurun_out/plain_tf32_${R}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -c 1 \
    -o gpurun_out/prof_gemm_tf32_${R} python tools/tf32_time.py > gpurun_out/ncu_tf32_${R}.log 2>&1
echo "tf32 full rc=$?"
