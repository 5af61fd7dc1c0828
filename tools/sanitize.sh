#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over smoke(): the tiny config through every
# ABI call (prefill, decode with drift, free, recycle) compared with the oracle after each call
mkdir -p gpurun_out
make -j16 > /dev/null 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|smoke ok' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
# NEXT-2: the attention kernel (shared-memory staging areas reused for page partials) on the tiny and the
# multi-page parity cases
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_attention.py -x -q -k "tiny or multi_page_d128" > gpurun_out/sanitize_attend_$tool.log 2>&1
  echo "attend $tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_attend_$tool.log | tr '\n' ' ')"
done
# the host-buffer decode step (library copy stream + events) and both classify instantiations
for tool in memcheck racecheck synccheck; do
  DKV_CD_LONG=${DKV_CD_LONG_SAN:-100} timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_host_step.py -x -q > gpurun_out/sanitize_host_step_$tool.log 2>&1
  echo "host step $tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_host_step_$tool.log | tr '\n' ' ')"
done
