#!/bin/bash
# One GPU call: pytest -m gpu, then the experiment tools (configs[3] grid + layers, N1 search
# tables, N4 synthetic networks, configs[4] VGG-16).  Usage: bash tools/gpu_suite.sh TAG
set -u
R=${1:-x}
O=gpurun_out/r02
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu_${R}.log 2>&1; echo "pytest rc=$?"
timeout 900 python tools/cfg4_grid.py > $O/cfg4_${R}.json 2> $O/cfg4_${R}.err; echo "cfg4 rc=$?"
timeout 900 python tools/search_tables.py > $O/search_${R}.json 2> $O/search_${R}.err; echo "search rc=$?"
timeout 900 python tools/synthetic_nets.py > $O/nets_${R}.json 2> $O/nets_${R}.err; echo "nets rc=$?"
timeout 900 python tools/vgg16.py > $O/vgg16_${R}.json 2> $O/vgg16_${R}.err; echo "vgg rc=$?"
