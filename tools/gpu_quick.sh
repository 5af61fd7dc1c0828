#!/bin/bash
# quick GPU iteration: build, GPU parity tests, one brief bench line (tools/bench_brief.sh args)
mkdir -p gpurun_out
make -j16 > gpurun_out/build_quick.log 2>&1 || { tail -30 gpurun_out/build_quick.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
bash tools/bench_brief.sh "$@"
