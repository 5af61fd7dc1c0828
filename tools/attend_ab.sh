#!/bin/bash
# A/B of attention build variants: tools/attend_ab.sh "EXTRA flags A" "EXTRA flags B" ...
mkdir -p gpurun_out
for v in "$@"; do
  echo "== variant: $v"
  make clean > /dev/null; make -j16 EXTRA="$v" > gpurun_out/build_ab.log 2>&1 || { tail -20 gpurun_out/build_ab.log; continue; }
  bash tools/attend_quick.sh
done
