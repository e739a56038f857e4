#!/bin/bash
# ncu --set full captures of the configs[1] sweep kernels (2D and 1D), after the same driver
# command exited 0 without ncu.  Usage (GPU box): bash tools/prof_sweep.sh TAG
set -u
R=${1:-r02}
mkdir -p gpurun_out/r02
python tools/prof_driver.py sweep > gpurun_out/r02/plain_sweep_${R}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'sweep2d_reg_kernel|sweep2d_kernel' -s 50 -c 1 \
    -o gpurun_out/r02/prof_sweep2d_${R} python tools/prof_driver.py sweep > gpurun_out/r02/ncu_sweep2d_${R}.log 2>&1
echo "sweep2d rc=$?"
ncu --set full --clock-control none --import-source on -k regex:sweep1d_kernel -s 50 -c 1 \
    -o gpurun_out/r02/prof_sweep1d_${R} python tools/prof_driver.py sweep > gpurun_out/r02/ncu_sweep1d_${R}.log 2>&1
echo "sweep1d rc=$?"
