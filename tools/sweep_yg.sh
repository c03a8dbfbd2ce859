# K4 (k_yg) sweep: L2 prefetch of B before the PDL wait, K3 early trigger, grid cap
# usage: bash tools/sweep_yg.sh "<config>:<pf bytes>:<sel_early>:<grid cap> ..."
for it in $1; do
  IFS=: read cfg pf early grid <<< "$it"
  export AXB_YG_PF=$pf AXB_SEL_EARLY=$early AXB_YG_GRID=$grid
  st=2000; [ $cfg = 5 ] && st=100
  timeout 300 python bench.py --config $cfg --steps $st --warmup 10 --no-cpu-baseline --no-e2e --no-tol 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('config $cfg pf=$pf early=$early grid=$grid', d['value'], d['ms_per_step'], r['k2_ms'], r['frac'], r['in_pipeline_ms'], d['clocks']['sm_mhz'])"
done
