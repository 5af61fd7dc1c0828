#!/bin/bash
for FL in "-DDKV_TC_SPLIT=0" "-DDKV_TC_SPLIT=1"; do
  rm -f build/k_attend_tc.o; make -j16 EXTRA="$FL" > /dev/null 2>&1
  echo "[$FL]"; timeout 600 python tools/tc_split_ab.py 2>&1 | tail -4
done
rm -f build/k_attend_tc.o; make -j16 > /dev/null 2>&1
