#!/bin/bash
# GPU-box driver for the round-2 ncu captures of the current kernels (one process, one GPU each):
#   bash profiles/gpu_prof.sh TAG [which...]   which: cfg4 split fp32 cfg3 tf32 cdcpred (default: cfg4 split fp32 cfg3 tf32)
# Writes gpurun_out/TAG_<which>.ncu-rep plus the raw and source pages as CSV (read here with summarize.py).
T=${1:-prof}; shift
W=${@:-cfg4 split fp32 cfg3 tf32}
O=gpurun_out
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on --target-processes application-only"
for w in $W; do
  case $w in
    cfg4)  K=regex:ann_tc_step_kernel;  CMD="python profiles/ann_probe.py cfg4 bf16 20000000 1" ;;
    split) K=regex:ann_tc_step_kernel;  CMD="python profiles/ann_probe.py cfg1 split 10000000 1" ;;
    tf32)  K=regex:ann_tc_step_kernel;  CMD="python profiles/ann_probe.py cfg1 tf32 10000000 1" ;;
    fp32)  K=regex:ann_f32; CMD="python profiles/ann_probe.py cfg1 fp32 4000000 1" ;;
    cfg3)  K=regex:exact_full4_kernel;  CMD="python profiles/exact_probe.py 50000000 1" ;;
    cdcpred) K=regex:cdc_pred_fused;    CMD="python profiles/cdc_probe.py 20000000 pred 1" ;;
    cdcstep) K=regex:cdc_step_kernel;   CMD="python profiles/cdc_probe.py 20000000 quantile" ;;
    cdchist) K=regex:cdc_hist_kernel;   CMD="python profiles/cdc_probe.py 100000000 quantile" ;;
  esac
  timeout 600 $NCU -k $K -s 1 -c 1 -o $O/${T}_$w -f $CMD > $O/${T}_$w.log 2>&1
  echo "$w ncu rc=$?"
  ncu -i $O/${T}_$w.ncu-rep --page raw --csv > $O/${T}_$w.raw.csv 2>/dev/null
  ncu -i $O/${T}_$w.ncu-rep --page source --csv --print-source sass > $O/${T}_$w.sass.csv 2>/dev/null
  ls -la $O/${T}_$w.*
done
