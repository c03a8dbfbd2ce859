"""GPU: every execution path under the bounds-checked build (the substitute for
compute-sanitizer, which the GPU pool does not allow).

libaxb_b200_checked.so (build.py --checked, -DAXB_CHECKED) checks the iteration
kernels' indexing — selected rows, streamed / combined rows of the TMA rings,
greedy group slots, CSR column indices, the scattered Gram row, trace and replay
slots, the sharded pack — and a violation fails the next call.  Each case of
tools/sanitize_cases.py (latency, general and batched persistent bodies, the
graph path with the TMA and the register K2, the sharded path, CSR operands, F2,
checkpoints) must run clean.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = ["lat", "general", "graph_tma", "graph_reg", "batch", "sharded", "sparse", "analysis",
         "checkpoint"]


@pytest.mark.parametrize("case", CASES)
def test_case_clean_under_bounds_checks(case):
    lib = os.path.join(ROOT, "paper_2408_05444_b200", "libaxb_b200_checked.so")
    if not os.path.exists(lib):
        pytest.skip("checked build absent")
    env = dict(os.environ, AXB_LIB_VARIANT="checked")
    code = ("import sys, runpy; sys.argv = ['sanitize_cases.py', '--case', %r]; "
            "import paper_2408_05444_b200._lib as L; assert L.load().axb_checked_build() == 1; "
            "runpy.run_path(%r, run_name='__main__')" % (case, os.path.join(ROOT, "tools",
                                                                              "sanitize_cases.py")))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr[-3000:]
    assert f"{case} ok" in out.stdout
