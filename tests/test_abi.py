"""CPU: the C-ABI library loads and exports every symbol include/axb_b200.h declares;
host-side API behaviour that needs no device (no compute calls here)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "axb_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(axb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2408_05444_b200 import _lib

    lib = C.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 38
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, f"declared but not exported: {missing}"
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(syms) <= bound, f"not bound in _lib.SIGNATURES: {set(syms) - bound}"
    assert _lib.load().axb_abi_version() == 1


def test_library_is_sm100a_only():
    """The product .so carries sm_100a SASS (no PTX JIT / other-arch fallback)."""
    import shutil
    import subprocess

    from paper_2408_05444_b200 import _lib

    cuobj = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobj):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobj, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_options_defaults_and_struct_layouts():
    from paper_2408_05444_b200 import _lib

    o = _lib.AxbOptions()
    _lib.load().axb_options_default(C.byref(o))
    assert (o.cache_gram, o.spectral_on_device, o.tie_guard, o.world_size) == (-1, -1, 1, 1)
    assert C.sizeof(_lib.AxbConfig) == 80 and C.sizeof(_lib.AxbReport) == 88
    assert C.sizeof(_lib.AxbOptions) == 80 and o.sm_share == 0


def test_no_device_fails_loudly():
    import paper_2408_05444_b200 as axb

    if axb.device_available():
        pytest.skip("a device is present")
    with pytest.raises(axb.CudaError, match="no CPU fallback"):
        axb.Solver(np.eye(2), np.eye(2), np.eye(2), None, axb.SolveConfig())


def test_method_validation_mirrors_reference():
    """test_solver.cpp:26-35."""
    import paper_2408_05444_b200 as axb

    with pytest.raises(axb.ConfigError):
        axb.Method.rgrbk(0.0).validate()
    with pytest.raises(axb.ConfigError):
        axb.Method.rgrbk(1.0).validate()
    bad = axb.Method.grbk()
    bad.theta = 0.3
    with pytest.raises(axb.ConfigError):
        bad.validate()
    axb.Method.rgrbk(0.5).validate()
    with pytest.raises(axb.ConfigError):
        axb.Method.parse("nope")
    assert axb.Method.parse("mwrbk").tag == axb.MethodTag.MWRBK
    assert axb.Method.parse("rgrbk", 0.3).label() == "rgrbk"


def test_trace_decimation():
    """test_solver.cpp:397-403."""
    import paper_2408_05444_b200 as axb

    assert axb.trace_point_due(0) and axb.trace_point_due(9999) and axb.trace_point_due(10000)
    assert not axb.trace_point_due(10001) and axb.trace_point_due(10010)


def test_error_taxonomy_codes():
    from paper_2408_05444_b200 import errors

    for code, cls in [(1, errors.ShapeError), (2, errors.DomainError), (3, errors.ConfigError),
                      (4, errors.DivergenceError), (5, errors.InvariantError),
                      (6, errors.ConvergenceError), (7, errors.CudaError),
                      (8, errors.CapacityError)]:
        with pytest.raises(cls):
            errors.raise_status(code, "x")
    with pytest.raises(errors.DivergenceError) as e:
        errors.raise_status(4, "d", iteration=12, residual_norm=3.5)
    assert e.value.iteration == 12 and e.value.residual_norm == 3.5


def build_cpp_example(tmp_path):
    import shutil
    import subprocess

    from paper_2408_05444_b200 import _lib

    gxx = shutil.which("g++")
    if not gxx:
        pytest.skip("g++ not available")
    exe = str(tmp_path / "dropin")
    src = os.path.join(ROOT, "tests", "cpp", "dropin_example.cpp")
    libdir = os.path.dirname(_lib.LIB_PATH)
    cmd = [gxx, "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", exe,
           f"-L{libdir}", "-laxb_b200", f"-Wl,-rpath,{libdir}"]
    subprocess.run(cmd, check=True)
    return exe


def test_cpp_dropin_header_compiles_and_fails_loudly_without_device(tmp_path):
    """include/axb_b200/solver.hpp compiles against the C-ABI; with no device the
    solver constructor throws (no CPU fallback)."""
    import subprocess

    import paper_2408_05444_b200 as axb

    exe = build_cpp_example(tmp_path)
    if axb.device_available():
        pytest.skip("device present: covered by the GPU test")
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 3 and "CudaError" in out.stdout, out.stdout


def test_csr_validation_errors_before_any_device_work():
    """SparseMatrix::validate (matrix.hpp:94-175) equivalents are host-side."""
    import scipy.sparse as sp

    import paper_2408_05444_b200 as axb

    bad = sp.csr_matrix(np.eye(3))
    bad.data[1] = 0.0  # stored zero: the reference rejects it
    with pytest.raises(axb.DomainError):
        axb.Solver(bad, np.eye(3), np.eye(3), None, axb.SolveConfig())
    nanm = sp.csr_matrix(np.eye(3))
    nanm.data[0] = np.nan
    with pytest.raises(axb.DomainError):
        axb.Solver(nanm, np.eye(3), np.eye(3), None, axb.SolveConfig())


def test_reference_dropin_builds_against_reference_headers():
    """tests/cpp/reference_dropin.cpp — the shim with the reference's own headers on
    the include path (axb::Matrix / axb::SolveConfig in, axb::SolveReport out, the
    reference's exception types) — compiles and links; without a device it exits 3
    after its first create (no CPU fallback)."""
    import subprocess

    import __graft_entry__ as g
    import paper_2408_05444_b200 as axb

    if not os.path.isdir(os.path.join(g.REF_INC, "axb")):
        pytest.skip("reference headers absent (GPU box): the prebuilt binary is used there")
    g.build_reference_dropin()
    assert os.path.exists(g.DROPIN_EXE)
    if axb.device_available():
        pytest.skip("device present: tests/test_gpu_dropin.py runs it")
    out = subprocess.run([g.DROPIN_EXE], capture_output=True, text=True)
    assert out.returncode == 3 and "device none" in out.stdout, out.stdout
