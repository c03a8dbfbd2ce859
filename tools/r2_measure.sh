# round-2 measurement pass: config-5 literal budget, config-3 profile, sanitizer probe,
# literal-size CPU check of the x64 rule, persistent-body phase times (rebuilds the box-local lib last)
set -x
timeout 900 python bench.py --config 5 --steps 10000 --warmup 10 --no-cpu-baseline --no-e2e --no-tol --no-sub > gpurun_out/bench_c5_1e4.json 2> gpurun_out/bench_c5_1e4.err; echo c5_1e4_exit=$?
bash tools/gpu_profile_c3.sh
mkdir -p gpurun_out/c3; cp gpurun_out/bench.json gpurun_out/bench_ref.json gpurun_out/launches.csv gpurun_out/c3/ 2>/dev/null
timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 99 python tools/sanitize_cases.py --case lat > gpurun_out/sanitize_probe.log 2>&1; echo sanitize_exit=$?; tail -5 gpurun_out/sanitize_probe.log
timeout 1500 python tools/config5_cpu_literal.py > gpurun_out/config5_cpu_literal.json 2> gpurun_out/config5_cpu_literal.err; echo literal_exit=$?; tail -2 gpurun_out/config5_cpu_literal.err
bash tools/persist_trace.sh > gpurun_out/persist_trace.txt 2>&1; echo persist_exit=$?
