"""Per-phase time of the persistent small-system kernel (build with -DAXB_TRACE_PERSIST).

usage: python tools/persist_timing.py   (env AXB_PERSIST_CLUSTER / AXB_PERSIST_GRID select the layout)
"""
import ctypes as C, os, sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle_lib as O, configs
import paper_2408_05444_b200 as axb
from paper_2408_05444_b200 import _lib
lib = _lib.load()
orc = O.oracle()
cases = {"config1": O.generate(orc, 7, 500, 100, 80, 400)[:4]}
A2, B2, X2, C2 = configs.config2(seed=2); cases["config2"] = (A2, B2, X2, C2)
cases["tall"] = O.generate(orc, 3, 8192, 64, 32, 96)[:4]
import scipy.sparse as sp
A4, B4, X4, C4 = configs.config4_channel(seed=4, nn=1024, half_band=7)
cases["config4"] = (A4, B4, X4, C4)
cases["config4csr"] = (sp.csr_matrix(A4), sp.csr_matrix(B4), X4, C4)
names = ["select", "y", "z1+X", "z2|pick", "R", "finalize", "barriers"]
methods = {"grbk": axb.Method.grbk(), "mwrbk": axb.Method.mwrbk(), "rbk": axb.Method.rbk()}
runs = ([("config1", mt) for mt in methods] + [("config2", "grbk"), ("config2", "mwrbk"), ("tall", "grbk"),
                                               ("config4", "grbk"), ("config4csr", "grbk"),
                                               ("config4:rr", "grbk"), ("config4csr:rr", "grbk")])
for name, mt in runs:
    A, B, X, Cm = cases[name.split(":")[0]]
    # ":rr" = the bench's fixed-budget stop (residual_rel): no X_ref, so no error tracking
    stop = axb.StopRule.residual_rel(0.0) if name.endswith(":rr") else axb.StopRule.solution_rrn(0.0, X)
    cfg = axb.SolveConfig(method=methods[mt], stop=stop, seed=42, refresh_interval=0)
    s = axb.Solver(A, B, Cm, None, cfg, axb.Options(spectral_max_iter=200000))
    s.steps(50); s.steps(2000)
    d = (C.c_uint64 * 8)(); lib.axb_solver_debug_state(s._h, d)
    it = max(1, d[7])
    parts = " ".join(f"{nm}={d[i] / it / 1e3:.2f}" for i, nm in enumerate(names))
    print(f"{name} {mt} lat={os.environ.get('AXB_PERSIST_LAT', 'auto')} grid={os.environ.get('AXB_PERSIST_GRID', 'auto')}: "
          f"{s.last_timing()['loop_ms'] / 2000 * 1e3:.2f} us/it; per-iteration us: {parts} (its {d[7]})")
