set -x
python - <<'PY'
import subprocess, os
from paper_2408_05444_b200 import build as b
cmd = [b.nvcc(), *b.NVCC_FLAGS, "-DAXB_TRACE_SELECT", "-shared", "-o", b.OUT,
       *[os.path.join(b.CSRC, s) for s in b.SOURCES], "-ldl"]
subprocess.run(cmd, check=True)
PY
timeout 300 python tools/sel_timing.py 3 2>&1 | grep -v Warn
