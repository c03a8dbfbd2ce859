# rebuild with per-phase stamps (box-local copy) and time the batched kernel's phases
python - <<'PY'
import subprocess, os
from paper_2408_05444_b200 import build as b
cmd = [b.nvcc(), *b.NVCC_FLAGS, "-DAXB_TRACE_PERSIST", "-shared", "-o", b.OUT,
       *[os.path.join(b.CSRC, s) for s in b.SOURCES], "-ldl"]
subprocess.run(cmd, check=True)
PY
timeout 300 python tools/batch_timing.py 148 2>&1 | grep -v Warn
timeout 300 python tools/batch_timing.py 16 2>&1 | grep -v Warn
