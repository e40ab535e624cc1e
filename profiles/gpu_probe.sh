#!/bin/bash
# GPU-box driver for timings + ncu captures of the ANN kernels (commands recorded in profiles/README.md).
# usage: bash profiles/gpu_probe.sh TAG  (writes gpurun_out/TAG_*)
set -x
T=${1:-probe}
O=gpurun_out
mkdir -p $O
for w in cfg1 cfg2_ou cfg2_cir; do
  for p in bf16 tf32 split fp32; do
    n=20000000; [ $w = cfg1 ] && n=10000000
    timeout 300 python profiles/ann_probe.py $w $p $n 3 >> $O/${T}_timings.jsonl 2>>$O/${T}_err.log
  done
done
NCU="ncu --set full --clock-control none --import-source on --target-processes application-only"
timeout 600 $NCU -k regex:ann_tc_step_kernel -s 1 -c 1 -o $O/${T}_softplus_bf16 -f python profiles/ann_probe.py cfg2_ou bf16 5000000 1 > $O/${T}_ncu1.log 2>&1
timeout 600 $NCU -k regex:ann_tc_step_kernel -s 1 -c 1 -o $O/${T}_split_cfg1 -f python profiles/ann_probe.py cfg1 split 2000000 1 > $O/${T}_ncu2.log 2>&1
timeout 600 $NCU -k regex:ann_tc_step_kernel -s 1 -c 1 -o $O/${T}_tf32_cfg1 -f python profiles/ann_probe.py cfg1 tf32 2000000 1 > $O/${T}_ncu3.log 2>&1
