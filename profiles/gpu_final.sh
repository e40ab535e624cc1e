#!/bin/bash
# GPU-box driver for a round's committed evidence: the default bench line, the launch list of the same
# command, the torchrun/NCCL launch path at world size 1, the reference arm, the pipe microbenchmarks and
# an ncu capture of the cfg3 FULL kernel.   usage: bash profiles/gpu_final.sh TAG
T=${1:-final}
O=gpurun_out
mkdir -p $O
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 2 --warmup 3 --no-modes --no-cpu-baseline > $O/${T}_torchrun.json 2> $O/${T}_torchrun.err
echo "torchrun rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/${T}_reference.json 2> $O/${T}_reference.err
echo "reference rc=$?"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipes_bench tests/native/pipes_bench.cu && \
  timeout 300 /tmp/pipes_bench > $O/${T}_pipes.txt 2>&1; echo "pipes rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --target-processes application-only --csv \
  --log-file $O/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/${T}_ncu_launch.log 2>&1
echo "launch list rc=$?"
bash profiles/gpu_prof.sh ${T} cfg3 > $O/${T}_prof.log 2>&1; grep rc= $O/${T}_prof.log
