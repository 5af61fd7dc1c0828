for FL in "-DDKV_CD_KCV_LONG=16" "-DDKV_CD_KCV_LONG=8" "-DDKV_CD_KCV_LONG=24"; do
  rm -f build/k_classify_decode.o; make -j16 EXTRA="$FL" > /dev/null 2>&1
  echo "[$FL]"; timeout 900 python tools/bench_configs.py qwen32b_thinking llama70b_shard8 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(' ', d['config'], d['decode_us']['classify_scan'])
"
done
rm -f build/k_classify_decode.o; make -j16 > /dev/null 2>&1
