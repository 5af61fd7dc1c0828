#!/bin/bash
# sweep the bulk writer's staging depth / CTAs-per-SM bound (compile-time) and time each build
for cfg in ${SWEEP:-"2 4" "1 4" "1 6" "2 3" "2 4"}; do
  set -- $cfg
  make -B -j16 EXTRA="-DDKV_BULK_STAGES=$1 -DDKV_BULK_MINB=$2" > /dev/null 2>&1 || { echo "build failed $cfg"; continue; }
  regs=$(grep -A2 "quant_prefill_kernelILi128ELi3" build/k_bulk.ptxas.log | grep -o "Used [0-9]* registers")
  echo "stages=$1 minb=$2 ($regs): $(python bench.py --steps 6 --warmup 3 --no-cpu-baseline --next2 0 2>&1 | tail -1 | python -c 'import json,sys; j=json.loads(sys.stdin.read()); q=j["quant_write"]; print(q["ms"], q["gbs"], q["frac_of_hbm_peak"])')"
done
make -B -j16 > /dev/null 2>&1
