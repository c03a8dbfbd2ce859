# K2 sweep with repeats (config 3): CTAs/SM × stages × tile × z staging [× carveout]
for cfg in "2 4 1024 1 x" "2 4 1024 1 x" "2 4 2048 0 x" "2 4 2048 0 x" "1 6 2048 1 x" "1 6 2048 1 x" "2 4 1024 1 100" "2 4 2048 0 100" "2 3 2048 1 x" "2 3 2048 1 x"; do
  set -- $cfg
  if [ "$5" = "x" ]; then unset AXB_CARVEOUT; else export AXB_CARVEOUT=$5; fi
  AXB_R_CPS=$1 AXB_R_STAGES=$2 AXB_R_TILE=$3 AXB_R_ZSTAGE=$4 timeout 120 python bench.py --steps 2000 --warmup 10 --no-cpu-baseline --no-e2e --no-tol 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cps=$1 stages=$2 tile=$3 z=$4 co=$5', d['value'], r['k2_ms'], r['frac'], d['clocks'])"
done
