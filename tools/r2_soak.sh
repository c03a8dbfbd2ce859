# round-2 soak on the final build: long randomised sweeps (new seeds), config 3's family to
# tolerance, the benchmark pool (F3) and the device reference solutions (F2)
set -x
O=gpurun_out/soak; mkdir -p $O
timeout 2400 python tools/fuzz_shapes.py 150 31 > $O/fuzz_shapes_seed31.txt 2>&1; echo shapes=$?; tail -1 $O/fuzz_shapes_seed31.txt
timeout 900 python tools/fuzz_run.py 60 32 > $O/fuzz_run_seed32.txt 2>&1; echo run=$?; tail -1 $O/fuzz_run_seed32.txt
timeout 900 python tools/fuzz_shard.py 60 33 > $O/fuzz_shard_seed33.txt 2>&1; echo shard=$?; tail -1 $O/fuzz_shard_seed33.txt
timeout 900 python tools/bench_pool.py --problems 2 --trials 60 > $O/pool_config1.json 2> $O/pool.err; echo pool=$?; tail -c 600 $O/pool_config1.json
timeout 900 python tools/bench_refsol.py > $O/refsol.json 2> $O/refsol.err; echo refsol=$?; tail -c 600 $O/refsol.json
timeout 1500 python tools/ttt_config3_family.py > $O/config3_family.jsonl 2> $O/family.err; echo family=$?; cut -c1-300 $O/config3_family.jsonl
