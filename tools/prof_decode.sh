#!/bin/bash
# ncu --set full of the three decode-step kernels (one launch each), for env settings given as args
TAG=${1:-x}
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"classify_decode|compact_alloc|quant_decode" -s 9 -c 3 -o gpurun_out/prof_decode_$TAG python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/prof_decode_$TAG.log 2>&1
