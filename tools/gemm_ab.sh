# K1 A/B: TMA-fed vs cp.async-fed DMMA GEMM (tests, pure GEMMs, checkpoints)
set -x
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/gemm_test.log 2>&1; echo test_exit=$?; tail -5 gpurun_out/gemm_test.log
for t in 1 0; do
  AXB_GEMM_TMA=$t timeout 600 python tools/bench_gemm.py pure > gpurun_out/gemm_pure_tma$t.log 2>&1; echo pure$t=$?
  AXB_GEMM_TMA=$t timeout 600 python tools/bench_gemm.py 3 > gpurun_out/gemm_ckpt3_tma$t.log 2>&1; echo ckpt$t=$?
done
cat gpurun_out/gemm_pure_tma*.log gpurun_out/gemm_ckpt3_tma*.log
