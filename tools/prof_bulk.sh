#!/bin/bash
TAG=${1:-x}
mkdir -p gpurun_out
for pf in 0 1; do
DKV_BULK_PF=$pf timeout 600 ncu --set full --import-source on --clock-control none -k regex:quant_prefill -s 1 -c 1 -o gpurun_out/prof_bulk_${TAG}_pf$pf python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof_bulk_${TAG}_pf$pf.log 2>&1
done
ls gpurun_out
