#!/bin/bash
# attention iteration: build, NEXT-2 GPU parity tests, the bench's next2 numbers
mkdir -p gpurun_out
make -j16 > gpurun_out/build_att.log 2>&1 || { tail -30 gpurun_out/build_att.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -3
python bench.py --no-cpu-baseline --steps 5 --warmup 3 2>&1 | tail -1 | python -c "
import json,sys
j=json.loads(sys.stdin.read()); n=j['next2']
print('attend_us', n['attend_us'], 'GB/s', n['attend_gbs'], 'frac', n['attend_frac_of_hbm_peak'], 'cls_fused', n['classify_fused_us'], '| bulk', j['quant_write']['ms'])"
