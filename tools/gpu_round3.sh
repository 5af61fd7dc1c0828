#!/bin/bash
# One full measurement call: build, GPU tests, smoke, bench line (+ reference arm), ncu launch list, full captures of
# the bulk writer (bench), the three decode kernels at a steady-state decode step (tools/decode_only.py) and
# attend_tc.   usage: tools/gpu_round3.sh TAG [skip_tests]
TAG=${1:-r2}
mkdir -p gpurun_out
make -j16 > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/smi_$TAG.txt
if [ -z "$2" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$TAG.log
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1; echo "ref rc=$?"
K='regex:quant_prefill|classify_decode|compact_alloc|quant_decode|classify_prefill|finish_prefill|set_requests|init_kernel|recycle_kernel|attend'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench_$TAG.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:quant_prefill_kernel -s 1 -c 1 -o gpurun_out/prof_bulk_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline --next2 0 > gpurun_out/prof_bulk_$TAG.log 2>&1; echo "ncu bulk rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"classify_decode|compact_alloc|quant_decode" -s 27 -c 3 -o gpurun_out/prof_decode_$TAG python tools/decode_only.py --steps 11 > gpurun_out/prof_decode_$TAG.log 2>&1; echo "ncu decode rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attend_tc -s 1 -c 1 -o gpurun_out/prof_attend_tc_$TAG python tools/decode_only.py --steps 3 --attend tc > gpurun_out/prof_attend_tc_$TAG.log 2>&1; echo "ncu attend_tc rc=$?"
ls gpurun_out | grep $TAG
if [ -n "$CONFIGS" ]; then
  timeout 1500 python tools/bench_configs.py > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; echo "configs rc=$?"
fi
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/scatter_bench tools/scatter_bench.cu && timeout 300 gpurun_out/scatter_bench > gpurun_out/scatter_$TAG.log 2>&1; echo "scatter rc=$?"; cat gpurun_out/scatter_$TAG.log
