#!/bin/bash
# Round evidence on one B200 (run under gpurun from the repo root):
#   gpurun -- 'bash tools/evidence.sh r02'
# 1) pytest -m gpu + smoke, 2) bench lines (native, reference arm), 3) the ncu launch list of
# the bench command (after it exited 0 without ncu), 4) ncu --set full captures of the top
# kernels from tools/prof_driver.py (each after the same driver command exited 0 without
# ncu), 5) the experiment tools (configs[3] grid, VGG-16, N1 tables, N4 stacks, N2 timings).
set -u
R=${1:-r02}
O=gpurun_out/$R
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > $O/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv $CMD \
    > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
full() {   # name, kernel regex, prof_driver mode, launch-skip, launch-count
  python tools/prof_driver.py $3 > $O/plain_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"$2" -s $4 -c $5 \
      -o $O/prof_$1 python tools/prof_driver.py $3 > $O/ncu_$1.log 2>&1; echo "ncu $1 rc=$?"
  summarise $1
}
summarise() {   # the reports exceed gpurun's 64 MiB return limit: keep their text summaries
  python tools/ncu_summary.py $O/prof_$1.ncu-rep --stalls > $O/ncu_$1.txt 2>&1
  { echo; echo "# hot instructions (tools/ncu_hot.py)"; python tools/ncu_hot.py $O/prof_$1.ncu-rep 15; } >> $O/ncu_$1.txt 2>&1
  rm -f $O/prof_$1.ncu-rep
}
full sweep2d 'sweep2d_reg_kernel' sweep 50 1
full sweep1d 'sweep1d_kernel' sweep 50 1
full huffjit 'wino_huffjit' huff 20 1
full n10 'sweep2d_kernel' cfg4 5 1
full layer 'gemm_kernel|input_kernel|output_kernel' layer 3 3
full score 'score_kernel' score 0 1
python tools/vgg_layers.py --only 0 > $O/plain_smallc.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:smallc_kernel -s 3 -c 1 \
    -o $O/prof_smallc python tools/vgg_layers.py --only 0 > $O/ncu_smallc.log 2>&1; echo "ncu smallc rc=$?"
summarise smallc
timeout 600 python tools/vgg_layers.py > $O/vgg_layers.json 2> $O/vgg_layers.err; echo "vgg layers rc=$?"
WINO_FORCE_COLLECTIVES=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline \
    > $O/bench_nccl_one_rank.json 2> $O/bench_nccl_one_rank.err; echo "nccl one-rank bench rc=$?"
timeout 900 python tools/cfg4_grid.py > $O/cfg4_grid.json 2> $O/cfg4_grid.err; echo "cfg4 rc=$?"
timeout 900 python tools/vgg16.py > $O/vgg16.json 2> $O/vgg16.err; echo "vgg rc=$?"
timeout 900 python tools/huffman_time.py > $O/variants_time.json 2> $O/variants_time.err; echo "variants rc=$?"
timeout 900 python tools/tf32_time.py > $O/layer_time.json 2> $O/layer_time.err; echo "layer time rc=$?"
timeout 1200 python tools/search_tables.py > $O/search_tables.json 2> $O/search_tables.err; echo "search rc=$?"
timeout 1200 python tools/synthetic_nets.py > $O/synthetic_nets.json 2> $O/synthetic_nets.err; echo "nets rc=$?"
