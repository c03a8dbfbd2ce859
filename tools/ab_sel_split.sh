#!/bin/bash
# A/B of the split greedy pre-selection (k_sel_greedy) on configs 3 and 5
for c in 3 5; do for v in 0 1; do
  AXB_SEL_SPLIT=$v timeout 400 python bench.py --config $c --no-cpu-baseline --no-e2e --no-tol 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('config', $c, 'split', $v, d['value'], d['roofline']['in_pipeline_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done; done
