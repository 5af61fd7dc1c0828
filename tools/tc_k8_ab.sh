for FL in "-DDKV_TC_K8_BIASED=1" "-DDKV_TC_K8_BIASED=0"; do
  rm -f build/k_attend_tc.o; make -j16 EXTRA="$FL" > /dev/null 2>&1
  echo "[$FL] $(ONLY=tc timeout 600 python tools/attend_ab.py 2>&1 | tail -1)"
  timeout 600 python tools/tc_debug.py 2>&1 | grep -o "out max err [0-9.e+-]*\|probs max err: high [0-9.e+-]* low [0-9.e+-]*" | sort | tail -4
  timeout 900 python -m pytest tests/test_gpu_attention_tc.py -q -x 2>&1 | tail -1
done
rm -f build/k_attend_tc.o; make -j16 > /dev/null 2>&1
