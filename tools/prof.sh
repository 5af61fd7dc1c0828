#!/bin/bash
# usage: tools/prof.sh TAG   — ncu --set full captures of the hot kernels (one launch each) + launch list
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:quant_prefill -s 1 -c 1 -o gpurun_out/prof_bulk_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof_bulk_$TAG.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"classify_decode|compact_alloc|quant_decode" -s 9 -c 3 -o gpurun_out/prof_decode_$TAG python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/prof_decode_$TAG.log 2>&1
ls -la gpurun_out
