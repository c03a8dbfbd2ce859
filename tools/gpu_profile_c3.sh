# config-3 bench + launch list + ncu full of the iteration kernels, and the K1 GEMM capture
set -x
B3="python bench.py --config 3 --steps 2000 --warmup 10"
timeout 600 $B3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$?
timeout 600 python bench.py --config 3 --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_exit=$?
B="python bench.py --config 3 --steps 60 --warmup 3 --no-cpu-baseline --no-e2e --no-tol"
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_(yg|yg_tma|zx|r|r_tma|select|ctrl|sel_greedy)$' -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1; echo list_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_(r_tma|yg|yg_tma|zx)$' -s 30 -c 3 -o gpurun_out/prof_iter $B > gpurun_out/ncu_full.log 2>&1; echo full_exit=$?
timeout 300 python tools/bench_gemm.py 3 > gpurun_out/gemm_plain.log 2>&1; echo gemm_plain_exit=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dgemm -s 4 -c 1 -o gpurun_out/prof_gemm python tools/bench_gemm.py 3 > gpurun_out/ncu_gemm.log 2>&1; echo gemm_exit=$?
