#!/bin/bash
# GPU-box driver: bench line, launch list of the same command, ncu --set full of the headline kernel.
# usage: bash profiles/gpu_bench.sh TAG [bench args...]   (writes gpurun_out/TAG_*)
T=${1:-bench}; shift
O=gpurun_out
mkdir -p $O
timeout 1200 python bench.py "$@" > $O/${T}_bench.json 2> $O/${T}_bench.err
echo "bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --target-processes application-only --csv \
  --log-file $O/${T}_launches.csv python bench.py "$@" --no-cpu-baseline > $O/${T}_ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --target-processes application-only \
  -k regex:ann_tc_step_kernel -s 1 -c 1 -o $O/${T}_cfg4_kernel -f python profiles/ann_probe.py cfg4 bf16 100000000 1 \
  > $O/${T}_ncu_full.log 2>&1
echo "ncu full rc=$?"
