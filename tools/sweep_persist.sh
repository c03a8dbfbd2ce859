# persistent-body knobs on configs 2 and 4: bash tools/sweep_persist.sh "<config>:<VAR=val,...> ..."
for spec in $1; do
  cfg=${spec%%:*}; envs=${spec#*:}
  ( [ "$envs" != "-" ] && export $(echo $envs | tr ',' ' ');
    timeout 300 python bench.py --config $cfg --steps 2000 --no-cpu-baseline --no-e2e --no-tol 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('config $cfg $envs', d['value'], d['ms_per_step'])" )
done
