# K2 launch-geometry sweep (config 3): CTAs/SM × ring stages × tile columns
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for cfg in "2 4 2048" "2 6 2048" "3 4 2048" "1 8 2048" "2 3 4096" "3 3 4096" "4 3 2048" "4 4 1024" "2 8 1024" "3 6 1024" "1 6 4096"; do
  set -- $cfg
  AXB_R_CPS=$1 AXB_R_STAGES=$2 AXB_R_TILE=$3 timeout 120 python bench.py --steps 600 --warmup 10 --no-cpu-baseline --no-e2e --no-tol 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cps=$1 stages=$2 tile=$3', d['value'], r['k2_ms'], r['frac'])"
done
