#!/bin/bash
# One GPU call: build check, pytest -m gpu, bench line, ncu launch list of the bench command.
#   gpurun -- 'bash tools/gpu_base.sh TAG'
set -u
R=${1:-x}
O=gpurun_out/$R
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
echo "launch list rc=$?"
