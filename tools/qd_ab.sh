#!/bin/bash
# A/B of quant_decode build variants (two bench runs each): usage tools/qd_ab.sh "FLAGS_A" "FLAGS_B" ...
mkdir -p gpurun_out
for F in "$@"; do
  rm -rf build paper_2412_03131_b200/libdkv.so
  make -j16 EXTRA="$F" > gpurun_out/build_ab.log 2>&1 || { tail -20 gpurun_out/build_ab.log; exit 1; }
  for i in 1 2; do echo "[$F] $(python tools/decode_ab.py 2>&1 | tail -1)"; done
done
rm -rf build paper_2412_03131_b200/libdkv.so; make -j16 > /dev/null 2>&1
