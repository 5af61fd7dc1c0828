#!/bin/bash
# A/B of decode-classify variants at the headline config and at the tie-heavy Qwen-32B thinking shape
# usage: tools/classify_ab2.sh "EXTRA flags A" "EXTRA flags B" ...
mkdir -p gpurun_out
for v in "$@"; do
  echo "== variant: '$v'"
  make clean > /dev/null; make -j16 EXTRA="$v" > gpurun_out/build_ab.log 2>&1 || { tail -20 gpurun_out/build_ab.log; continue; }
  for i in 1 2; do timeout 600 bash tools/bench_brief.sh --next2 0 --steps 40; done
  timeout 900 python tools/bench_configs.py qwen32b_thinking 2>&1 | tail -1 | python -c "
import json,sys
j=json.loads(sys.stdin.read()); print('qwen32b_thinking', j['decode_us'])"
done
