#!/bin/bash
# brief bench summary (one line) — used during tuning
python bench.py --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "
import json,sys
j=json.loads(sys.stdin.read())
d=j['decode_step_us']; q=j['quant_write']
print(f\"compact={j['value']} p50={d['compact_alloc_p50']} floor={d.get('launch_floor')} p99={d['compact_alloc_p99']} classify={d['classify']} qw_dec={d['quant_write']} step={d['step']} | bulk {q['ms']}ms {q['gbs']}GB/s frac={q['frac_of_hbm_peak']} | cls_frac={j['roofline_decode']['frac']} e2e={j['e2e']['value']}\")"
