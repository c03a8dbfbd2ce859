# ncu of the config-1 persistent latency kernel (one 2000-iteration launch)
set -x
timeout 300 python tools/prof_small.py > gpurun_out/prof_small_plain.log 2>&1; cat gpurun_out/prof_small_plain.log | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_persist_lat' -s 1 -c 1 -o gpurun_out/prof_small python tools/prof_small.py > gpurun_out/prof_small_ncu.log 2>&1; echo ncu_exit=$?
