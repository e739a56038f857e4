#!/bin/bash
# One GPU call for the layer path: layer / VGG / TF32 GPU tests, layer timings (configs[2]
# bench leg, configs[3] layers, VGG-16 x64), ncu launch list of the VGG forward.
#   gpurun -- 'bash tools/gpu_layer.sh TAG'
set -u
R=${1:-x}
O=gpurun_out/$R
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_vgg.py tests/test_gpu_tf32.py tests/test_gpu_guard.py -q -x > $O/pytest_layer.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python tools/tf32_time.py > $O/layer_time.json 2> $O/layer_time.err; echo "layer time rc=$?"
timeout 900 python tools/vgg16.py --scored-batch 8 > $O/vgg16.json 2> $O/vgg16.err; echo "vgg rc=$?"
python tools/prof_driver.py vgg > $O/plain_vgg.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $O/launches_vgg.csv python tools/prof_driver.py vgg > $O/ncu_vgg.log 2>&1; echo "ncu vgg rc=$?"
