#!/bin/bash
# Jacobi round grid sweep at config-3 sizes (tools/bench_refsol.py, device ms)
for c in 148 296 384 592 1024; do
  echo -n "ctas=$c "; AXB_JACOBI_CTAS=$c timeout 300 python tools/bench_refsol.py --repeat 1 --sample 64x16 | python -c "import json,sys; d=json.load(sys.stdin); print(d['device_ms'], d['us_per_round'], d['sweeps'])"
done
echo -n "default "; timeout 300 python tools/bench_refsol.py --repeat 1 --sample 64x16 | python -c "import json,sys; d=json.load(sys.stdin); print(d['device_ms'], d['us_per_round'], d['sweeps'])"
