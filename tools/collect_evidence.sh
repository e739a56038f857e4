#!/bin/bash
# Copy the outputs of tools/evidence.sh TAG (merged back under gpurun_out/TAG) into profiles/
# under the round's names.  Usage: bash tools/collect_evidence.sh TAG [ROUND]
set -eu
O=gpurun_out/$1
R=${2:-r02}
P=profiles
cp $O/bench.json $P/${R}_bench.json
cp $O/bench_reference.json $P/${R}_bench_reference_arm.json
cp $O/launches_bench.csv $P/${R}_launches_bench.csv
python tools/launch_table.py $O/launches_bench.csv --families > $P/${R}_launches_bench_families.txt
for k in sweep2d sweep1d huffjit n10 layer score smallc; do cp $O/ncu_$k.txt $P/${R}_ncu_$k.txt; done
cp $O/cfg4_grid.json $P/${R}_cfg4_grid.json
cp $O/vgg16.json $P/${R}_vgg16.json
cp $O/vgg_layers.json $P/${R}_vgg_layers.json
[ -f $O/vgg_layers_unfused.json ] && cp $O/vgg_layers_unfused.json $P/${R}_vgg_layers_unfused_first_layer.json
[ -f $O/layer_ab.jsonl ] && cp $O/layer_ab.jsonl $P/${R}_layer_ab.jsonl
cp $O/variants_time.json $P/${R}_variants_sweep_time.json
cp $O/layer_time.json $P/${R}_layer_time.json
cp $O/search_tables.json $P/${R}_search_tables_huffman.json
cp $O/synthetic_nets.json $P/${R}_synthetic_nets_N4.json
cp $O/pytest_gpu.log $P/${R}_pytest_gpu.log
cp $O/smoke.log $P/${R}_smoke.log
grep -v "^NCCL version" $O/bench_nccl_one_rank.json > $P/${R}_bench_nccl_one_rank.json
python - "$O" <<'PY'
import json, re, sys
t = open(sys.argv[1] + "/ncu_sweep2d.txt").read()
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tot = 0.0
for k in ("read", "write"):
    m = re.search(r"dram__bytes_%s.sum\s+([\d.]+) (\w+)" % k, t)
    tot += float(m.group(1)) * unit[m.group(2)]
d = json.load(open("profiles/ncu_traffic.json"))
d["sweep2d_dram_bytes_per_launch"] = int(tot)
json.dump(d, open("profiles/ncu_traffic.json", "w"), indent=2)
PY
echo collected $O
