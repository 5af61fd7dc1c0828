#!/bin/bash
# A/B of decode-classify build variants: tools/classify_ab.sh "EXTRA flags A" "EXTRA flags B" ...
# each variant: clean build, then two brief bench lines (classify / compact / quant-write us, bulk GB/s)
mkdir -p gpurun_out
for v in "$@"; do
  echo "== variant: '$v'"
  make clean > /dev/null; make -j16 EXTRA="$v" > gpurun_out/build_ab.log 2>&1 || { tail -20 gpurun_out/build_ab.log; continue; }
  for i in 1 2; do timeout 600 bash tools/bench_brief.sh --next2 0 --steps 40; done
done
