# rebuild the library with per-phase stamps (box-local copy) and time the persistent bodies
set -x
python - <<'PY'
import subprocess, os
from paper_2408_05444_b200 import build as b
cmd = [b.nvcc(), *b.NVCC_FLAGS, "-DAXB_TRACE_PERSIST", "-shared", "-o", b.OUT,
       *[os.path.join(b.CSRC, s) for s in b.SOURCES], "-ldl"]
subprocess.run(cmd, check=True)
PY
for v in "AXB_PERSIST_LAT=0" "AXB_PERSIST_LAT=256"; do
  echo "== $v"; env $v timeout 300 python tools/persist_timing.py 2>&1 | grep -v Warn
done
