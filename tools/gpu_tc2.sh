#!/bin/bash
# TC attention + tier iteration: build, TC / tier / attention tests, the attention A/B probe, the config sweep
TAG=${1:-tc2}
mkdir -p gpurun_out
make -j16 > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_attention_tc.py tests/test_gpu_top_tier.py tests/test_gpu_attention.py -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python tools/attend_ab.py 2>&1 | tail -4
if [ -n "$CONFIGS" ]; then
  timeout 2000 python tools/bench_configs.py > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; echo "configs rc=$?"; tail -2 gpurun_out/configs_$TAG.err
fi
