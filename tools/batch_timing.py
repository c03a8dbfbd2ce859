"""Per-phase time of the batched small-system kernel (k_persist_batch, one CTA per
system; build with -DAXB_TRACE_PERSIST).  usage: python tools/batch_timing.py [n]"""
import ctypes as C, sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle_lib as O
import paper_2408_05444_b200 as axb
from paper_2408_05444_b200 import _lib
lib = _lib.load()
orc = O.oracle()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 148
A, B, X, Cm = O.generate(orc, 7, 500, 100, 80, 400)
names = ["select", "y", "z1+X", "z2|pick", "R", "finalize", "barriers"]
for mt, meth in (("grbk", axb.Method.grbk()), ("mwrbk", axb.Method.mwrbk())):
    hs = [axb.Solver(A, B, Cm, None, axb.SolveConfig(method=meth, stop=axb.StopRule.solution_rrn(0.0, X),
                                                     seed=t, max_iter=3000, refresh_interval=0))
          for t in range(n)]
    axb.run_many(hs)
    d = (C.c_uint64 * 8)()
    lib.axb_solver_debug_state(hs[0]._h, d)
    it = max(1, d[7])
    parts = " ".join(f"{nm}={d[i] / it / 1e3:.2f}" for i, nm in enumerate(names))
    print(f"batch of {n} config-1 {mt}: per-iteration us: {parts} (its {d[7]})", flush=True)
