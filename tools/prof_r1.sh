set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
K='regex:quant_prefill|classify_decode|compact_alloc|quant_decode|classify_prefill|finish_prefill|set_requests|init_kernel'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:quant_prefill -s 1 -c 1 -o gpurun_out/prof_bulk_r1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof_bulk.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"classify_decode|compact_alloc|quant_decode" -s 9 -c 3 -o gpurun_out/prof_decode_r1 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/prof_decode.log 2>&1
ls -la gpurun_out
