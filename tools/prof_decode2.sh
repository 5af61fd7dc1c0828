#!/bin/bash
# targeted ncu --set full captures of each decode kernel (a mid-run decode step) and of attend_tc
TAG=${1:-r2}
mkdir -p gpurun_out
make -j16 > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
for K in quant_decode compact_alloc classify_decode; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$K -s 9 -c 1 -o gpurun_out/prof_${K}_$TAG python tools/decode_only.py --steps 11 > gpurun_out/prof_${K}_$TAG.log 2>&1; echo "$K rc=$?"
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attend_tc -s 2 -c 1 -o gpurun_out/prof_attend_tc_$TAG python tools/decode_only.py --steps 4 --attend tc > gpurun_out/prof_attend_tc_$TAG.log 2>&1; echo "attend_tc rc=$?"
if [ -n "$2" ]; then
  time (timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1); echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_$TAG.json | cut -c1-400
fi
