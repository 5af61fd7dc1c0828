#!/bin/bash
# TC attention iteration: build, its tests, a bench line, one ncu --set full capture of attend_tc_kernel
TAG=${1:-tc}
mkdir -p gpurun_out
make -j16 > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_attention_tc.py tests/test_gpu_multi.py -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python - <<'PY'
import json,sys,os
tag=os.environ.get("TAG","tc")
PY
python -c "
import json
d=json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1])
print('value', d['value'], 'step', d['decode_step_us']['step'], 'qw', d['decode_step_us']['quant_write'])
print('graph', {k: d['graph'][k] for k in ('one_step_graph_us','graph_step_us','graph_step_us_no_pdl')} if d['graph'] else None)
print('exact attend', d['next2']['attend_us'], 'tc', d['next2']['tc']['attend_us'], d['next2']['tc']['roofline']['frac'], d['next2']['tc']['speedup_vs_fp16_roofline'])
"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attend_tc_kernel -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof_$TAG.log 2>&1; echo "ncu rc=$?"
