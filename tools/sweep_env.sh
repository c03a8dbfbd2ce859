# generic A/B sweep: bash tools/sweep_env.sh "<config>:<VAR=val,VAR=val> ..."  (use - for no env)
for spec in $1; do
  cfg=${spec%%:*}; envs=${spec#*:}
  st=2000; [ $cfg = 5 ] && st=100
  ( [ "$envs" != "-" ] && export $(echo $envs | tr ',' ' ');
    timeout 300 python bench.py --config $cfg --steps $st --warmup 10 --no-cpu-baseline --no-e2e --no-tol 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('config $cfg $envs', d['value'], d['ms_per_step'], r['k2_ms'], r['frac'], r['in_pipeline_ms'], d['clocks']['sm_mhz'])" )
done
