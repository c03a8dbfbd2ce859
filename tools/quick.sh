timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$?
python -c "
import json; d=json.load(open('gpurun_out/bench.json')); r=d['roofline']; print(d['value'], d['ms_per_step'], r['k2_ms'], r['frac'], r['k2_share_of_step'], d['e2e']['value'], d['time_to_tol'])"
