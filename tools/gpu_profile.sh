# GPU round trip: parity tests, default bench, reference arm, launch list, one ncu --set full capture.
set -x
timeout 1200 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo pytest_exit=$?; tail -3 gpurun_out/pytest.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_exit=$?
B="python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-tol"
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_(yg|yg_tma|zx|r|r_tma|select|ctrl|sel_greedy)$' -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1; echo list_exit=$?
timeout 300 $B > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_(r_tma|yg|yg_tma|zx)$' -s 20 -c 3 -o gpurun_out/prof_iter $B > gpurun_out/ncu_full.log 2>&1; echo full_exit=$?
