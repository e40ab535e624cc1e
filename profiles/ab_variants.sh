#!/bin/bash
# A/B timing of epilogue variants through the experiment build (SL7_LIB=libsl7_ab.so, SL7_TC_VARIANT=v).
# usage: bash profiles/ab_variants.sh WORKLOAD PREC N "v1 v2 ..."
W=$1; P=$2; N=$3
for v in $4; do
  echo -n "variant $v: "
  SL7_LIB=paper_2302_05170_b200/libsl7_ab.so SL7_TC_VARIANT=$v timeout 300 python profiles/ann_probe.py $W $P $N 3
done
