# latency body: loads in flight per lane (AXB_LAT_KU dots, AXB_LAT_KR row updates) vs spills;
# box-local rebuilds, configs 1 and 4 (one channel dense / CSR via tools/bench_config4.py)
for v in ${COMBOS:-8_4 6_4 5_4 4_4 3_4 8_2 6_2 4_3 4_6}; do set -- ${v/_/ }
python - <<PY
import subprocess, os
from paper_2408_05444_b200 import build as b
cmd = [b.nvcc(), *b.NVCC_FLAGS, "-DAXB_LAT_KU=$1", "-DAXB_LAT_KR=$2", "-shared", "-o", b.OUT,
       *[os.path.join(b.CSRC, s) for s in b.SOURCES], "-ldl"]
subprocess.run(cmd, check=True)
PY
echo "== KU=$1 KR=$2"
timeout 300 python bench.py --config 1 --no-cpu-baseline --no-e2e --no-tol 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('config 1', d['value'], d['ms_per_step'])"
timeout 300 python tools/bench_config4.py 2>&1 | grep "half-band 7"
done
