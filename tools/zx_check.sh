#!/bin/bash
# k_zx A/B: bench configs 5 and 3 (value, in-pipeline kernel ms) + ncu k_zx duration at config 5
for c in 5 3; do
  timeout 400 python bench.py --config $c 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['config']['workload'][:8], d['value'], d['roofline']['in_pipeline_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_zx|k_yg" -s 6 -c 4 python bench.py --config 5 --steps 3 --warmup 3 2>/dev/null | grep -E "k_zx|k_yg|duration|bytes" | head -24
