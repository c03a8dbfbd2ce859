# config 3 / config 5 whole-iteration rates (k_zx pipelining, carve-out incl. k_zx)
for st in 500 900; do
  timeout 120 python bench.py --config 3 --steps $st --warmup 10 --no-cpu-baseline --no-e2e --no-tol 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('config3 steps=$st', d['value'], r['in_pipeline_ms'], r['k2_ms'], r['frac'])"
done
timeout 200 python bench.py --config 5 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-tol 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('config5', d['value'], r['in_pipeline_ms'], r['k2_ms'], r['frac'])"
