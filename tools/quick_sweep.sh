#!/bin/bash
# Quick GPU iteration on the sweep kernels: bench line without the layer / cpu legs, then
# ncu --set full captures of the 2D and 1D configs[1] kernels.  Usage: bash tools/quick_sweep.sh TAG
set -u
R=${1:-x}
mkdir -p gpurun_out/r02
python bench.py --steps 5 --warmup 3 --no-layer --no-cpu-baseline > gpurun_out/r02/bench_${R}.json 2> gpurun_out/r02/bench_${R}.err
echo "bench rc=$?"
bash tools/prof_sweep.sh ${R}
