#!/bin/bash
# attend_tc iteration: build, TC tests, timing (tools/attend_ab.py), one ncu --set full capture of attend_tc_kernel
TAG=${1:-tcp}
mkdir -p gpurun_out
make -j32 > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest tests/test_gpu_attention_tc.py -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
fi
timeout 600 python tools/attend_ab.py 2>&1 | tail -1
ONLY=tc timeout 900 ncu --set full --import-source on --clock-control none -k regex:attend_tc_kernel -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/attend_ab.py > gpurun_out/prof_$TAG.log 2>&1; echo "ncu rc=$?"
