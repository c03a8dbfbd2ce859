timeout 300 python tools/bench_gemm.py 3 > gpurun_out/gemm_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dgemm -s 4 -c 1 -o gpurun_out/prof_gemm python tools/bench_gemm.py 3 > gpurun_out/ncu_gemm.log 2>&1; echo gemm_exit=$?
cat gpurun_out/gemm_plain.log
