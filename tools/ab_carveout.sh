# A/B: shared-memory carve-out (computed vs K2-only) on config 3 and 5, twice each
for rep in 1 2; do for co in auto 60; do
  if [ "$co" = auto ]; then unset AXB_CARVEOUT; else export AXB_CARVEOUT=$co; fi
  timeout 120 python bench.py --config 3 --steps 900 --warmup 10 --no-cpu-baseline --no-e2e --no-tol 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c3 co=$co', d['value'], r['in_pipeline_ms'])"
  timeout 200 python bench.py --config 5 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-tol 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c5 co=$co', d['value'], r['in_pipeline_ms'])"
done; done
