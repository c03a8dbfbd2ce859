# second soak on the final build (after the latency-body re-tuning): self-diagnosing sweeps, new seeds
set -x
O=gpurun_out/soak2; mkdir -p $O
timeout 3000 python tools/fuzz_shapes.py 240 41 > $O/fuzz_shapes_seed41.txt 2>&1; echo shapes=$?; tail -1 $O/fuzz_shapes_seed41.txt
timeout 900 python tools/fuzz_run.py 100 42 > $O/fuzz_run_seed42.txt 2>&1; echo run=$?; tail -1 $O/fuzz_run_seed42.txt
timeout 900 python tools/fuzz_shard.py 100 43 > $O/fuzz_shard_seed43.txt 2>&1; echo shard=$?; tail -1 $O/fuzz_shard_seed43.txt
