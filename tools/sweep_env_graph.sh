# Generic env sweep of the graph-path iteration (configs 3 and 5).
# usage: bash tools/sweep_env_graph.sh "<config>:<VAR=val[,VAR=val]> ..."   ("-" = defaults)
for it in $1; do
  cfg=${it%%:*}; envs=${it#*:}
  st=2000; [ $cfg = 5 ] && st=100
  ( [ "$envs" != "-" ] && for kv in ${envs//,/ }; do export "$kv"; done
    timeout 300 python bench.py --config $cfg --steps $st --warmup 10 --no-cpu-baseline --no-e2e --no-tol 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('config $cfg $envs', d['value'], d['ms_per_step'], r['k2_ms'], r['in_pipeline_ms'], d['clocks']['sm_mhz'])" )
done
