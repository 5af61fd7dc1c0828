#!/bin/bash
# attend_tc build-knob A/B: for each "FLAGS" argument, rebuild k_attend_tc.o with them, time configs[1] attention
# (tools/attend_ab.py, tensor-core path only); the default build is restored at the end.
mkdir -p gpurun_out
for FL in "$@"; do
  rm -f build/k_attend_tc.o
  make -j16 EXTRA="$FL" > gpurun_out/tc_ab_build.log 2>&1 || { tail -20 gpurun_out/tc_ab_build.log; continue; }
  echo "[$FL] $(ONLY=tc timeout 600 python tools/attend_ab.py 2>&1 | tail -1)"
done
rm -f build/k_attend_tc.o; make -j16 > /dev/null 2>&1
