#!/bin/bash
# ncu --set full of the three decode-step kernels of the 2nd decode step (bench --steps 2 --warmup 1:
# 3 bulk rounds contribute 9 filtered launches before the decode phase, then 3 per step)
TAG=${1:-x}
mkdir -p gpurun_out
make -j16 > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"classify_decode|compact_alloc|quant_decode" -s 12 -c 3 -o gpurun_out/prof_decode_$TAG python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/prof_decode_$TAG.log 2>&1
echo "ncu rc=$?"
