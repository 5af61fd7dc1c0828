#!/bin/bash
# A/B of build variants.  Every variant: attend_tc vs exact (tools/attend_ab.py at configs[1]).  Prefixes:
#   CD: also the decode classify scan at the tie-heavy Llama-3-70B shard (tools/bench_configs.py llama70b_shard8)
#   BB: also two brief bench lines (decode step kernels, no NEXT-2 / graph phases)
# usage: tools/ab_tc_cd.sh "BB:CD:EXTRA flags A" "EXTRA flags B" ...
mkdir -p gpurun_out
for v in "$@"; do
  cd_run=0; bb_run=0
  while true; do
    if [[ "$v" == CD:* ]]; then cd_run=1; v="${v#CD:}";
    elif [[ "$v" == BB:* ]]; then bb_run=1; v="${v#BB:}";
    else break; fi
  done
  echo "== variant: '$v'"
  make clean > /dev/null; make -j32 EXTRA="$v" > gpurun_out/build_ab.log 2>&1 || { tail -20 gpurun_out/build_ab.log; continue; }
  timeout 600 python tools/attend_ab.py 2>&1 | tail -1
  if [ $bb_run = 1 ]; then
    for i in 1 2; do timeout 600 bash tools/bench_brief.sh --next2 0 --steps 40; done
  fi
  if [ $cd_run = 1 ]; then
    timeout 900 python tools/bench_configs.py llama70b_shard8 2>&1 | tail -1 | python -c "
import json,sys
j=json.loads(sys.stdin.read()); print('llama70b_shard8', j['decode_us'], j['attend_ms'], j['attend_tc_ms'])"
  fi
done
make clean > /dev/null; make -j32 > /dev/null 2>&1
