# z row-chunk sweep on the persistent bodies (configs 2, 4; batched config-1 pool)
for j in 128 64 32 16; do
  export AXB_Z_JROWS=$j
  for c in 2 4; do
    timeout 300 python bench.py --config $c --steps 2000 --no-cpu-baseline --no-e2e --no-tol 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('jrows $j config $c', d['value'], d['ms_per_step'])"
  done
  echo "jrows $j pool: $(timeout 300 python tools/prof_batch.py 148 2>/dev/null | tail -1)"
done
