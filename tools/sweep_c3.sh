# config 3: whole-iteration rate per k_zx row chunk and greedy-select split
for jr in 32 64 128 256; do for ss in 0 1; do
  AXB_Z_JROWS=$jr AXB_SEL_SPLIT=$ss timeout 120 python bench.py --config 3 --steps 2000 --warmup 10 --no-cpu-baseline --no-e2e --no-tol 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('jrows=$jr split=$ss', d['value'], r['in_pipeline_ms'], r['k2_ms'])"
done; done
B="python bench.py --config 3 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-tol"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_(yg|zx)$' -s 20 -c 2 -o gpurun_out/prof_c3 $B > gpurun_out/ncu_c3.log 2>&1; echo full=$?
