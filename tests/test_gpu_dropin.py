"""GPU: the reference's own call sites through the C++ shim.

tools/bin/reference_dropin is tests/cpp/reference_dropin.cpp compiled against the
unmodified reference headers (/root/reference/proj/include, by
__graft_entry__.build() in the build container) and the shim
include/axb_b200/solver.hpp over libaxb_b200.so.  It runs acceptance.cpp:128-141's
step() loop in lockstep on axb::Solver and axb_b200::Solver (same row each step,
X within 1e-10 at the same k), axb_b200::solve(const axb::Matrix&, …) on CSR and
dense operands against axb::solve (solver.hpp:518-532), and the reference's
exception types (axb::ShapeError, axb::ConfigError).
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tools", "bin", "reference_dropin")


def test_reference_call_sites_through_the_shim():
    if not os.path.exists(EXE):
        import __graft_entry__ as g

        g.build_reference_dropin()
    if not os.path.exists(EXE):
        pytest.skip("tools/bin/reference_dropin not built (needs the reference headers)")
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ALL_OK" in out.stdout
    assert out.stdout.count(" ok ") >= 11
