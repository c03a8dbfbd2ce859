# round-2 parity refresh on the final build: randomised sweeps with new seeds and the
# full-size pins of configs 2, 4 and 5 (logs → gpurun_out/parity/)
set -x
O=gpurun_out/parity; mkdir -p $O
timeout 1200 python tools/fuzz_shapes.py 60 21 > $O/fuzz_shapes_seed21.txt 2>&1; echo shapes=$?; tail -2 $O/fuzz_shapes_seed21.txt
timeout 900 python tools/fuzz_run.py 30 22 > $O/fuzz_run_seed22.txt 2>&1; echo run=$?; tail -2 $O/fuzz_run_seed22.txt
timeout 900 python tools/fuzz_shard.py 40 23 > $O/fuzz_shard_seed23.txt 2>&1; echo shard=$?; tail -2 $O/fuzz_shard_seed23.txt
timeout 900 python tools/config2_sequence.py > $O/config2_sequence_1e4.jsonl 2> $O/config2_sequence.err; echo c2=$?; tail -2 $O/config2_sequence_1e4.jsonl | cut -c1-400
timeout 900 python tools/config4_parity.py > $O/config4_parity_full.jsonl 2> $O/config4_parity.err; echo c4=$?; tail -2 $O/config4_parity_full.jsonl | cut -c1-300
timeout 1200 python tools/config5_shard_invariance.py > $O/config5_shard_invariance.jsonl 2> $O/config5_shard.err; echo c5=$?; tail -2 $O/config5_shard_invariance.jsonl | cut -c1-400
