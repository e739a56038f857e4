#!/bin/bash
set -u
R=${1:-x}
O=gpurun_out/r02
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_vgg.py tests/test_gpu_tf32.py -q > $O/pytest_layer_${R}.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_${R}.json 2> $O/bench_${R}.err; echo "bench rc=$?"
timeout 900 python tools/vgg16.py > $O/vgg16_${R}.json 2> $O/vgg16_${R}.err; echo "vgg rc=$?"
python tools/prof_driver.py score > $O/plain_score_${R}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'score_kernel' -c 1 \
    -o $O/prof_score_${R} python tools/prof_driver.py score > $O/ncu_score_${R}.log 2>&1; echo "ncu score rc=$?"
python tools/prof_driver.py cfg4 > $O/plain_cfg4_${R}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'sweep2d' -s 2 -c 2 \
    -o $O/prof_cfg4_${R} python tools/prof_driver.py cfg4 > $O/ncu_cfg4_${R}.log 2>&1; echo "ncu cfg4 rc=$?"
