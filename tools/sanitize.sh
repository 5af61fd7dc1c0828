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
