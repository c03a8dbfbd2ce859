# config 3: bench line + launch list of the iteration kernels
set -x
timeout 600 python bench.py --config 3 --steps 500 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo b3=$?
B="python bench.py --config 3 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-tol"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_(yg|zx|r_tma|sel_greedy)$' -c 200 --csv --log-file gpurun_out/launches3.csv $B > gpurun_out/ncu3.log 2>&1; echo list=$?
