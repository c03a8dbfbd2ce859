# K2 row-grab granularity sweep (config 3 and the config-5 default)
# usage: bash tools/sweep_grab.sh "<config:grab> ..."
for cg in $1; do
  cfg=${cg%%:*}; g=${cg##*:}
  if [ "$g" = "auto" ]; then unset AXB_R_GRAB; else export AXB_R_GRAB=$g; fi
  st=2000; [ $cfg = 5 ] && st=100
  timeout 300 python bench.py --config $cfg --steps $st --warmup 10 --no-cpu-baseline --no-e2e --no-tol 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('config $cfg grab=$g', d['value'], r['k2_ms'], r['frac'], r['in_pipeline_ms'], d['clocks']['sm_mhz'])"
done
