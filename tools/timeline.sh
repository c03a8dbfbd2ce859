# rebuild the library with the timeline stamps (box-local copy) and print configs 3 and 5
set -x
python - <<'PY'
import subprocess, os
from paper_2408_05444_b200 import build as b
cmd = [b.nvcc(), *b.NVCC_FLAGS, "-DAXB_TRACE_TIMELINE", "-shared", "-o", b.OUT,
       *[os.path.join(b.CSRC, s) for s in b.SOURCES], "-ldl"]
subprocess.run(cmd, check=True)
PY
for c in ${@:-3 5}; do timeout 600 python tools/timeline.py $c 2>&1 | grep -v Warn | tee gpurun_out/timeline_config$c.txt; done
