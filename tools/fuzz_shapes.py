"""Randomised shape sweep against the oracle (robustness probe): every execution
path (latency body, general persistent body, graph path with the TMA or the
register-streaming K2, G cached or not) and every method.
usage: python tools/fuzz_shapes.py [cases] [seed] [only: comma-separated case numbers]
A case that leaves the oracle's rows is followed by a diagnosis line (tools/fuzz_diag.py)."""
import sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests"); sys.path.insert(0, "tools")
import numpy as np
import oracle_lib as O
import paper_2408_05444_b200 as axb
from fuzz_diag import diagnose

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
only = {int(x) for x in sys.argv[3].split(",")} if len(sys.argv) > 3 else None
orc = O.oracle()
meths = [(O.GRBK, None, axb.Method.grbk()), (O.MWRBK, None, axb.Method.mwrbk()),
         (O.RBK, None, axb.Method.rbk()), (O.BK, None, axb.Method.bk()),
         (O.RGRBK, 0.3, axb.Method.rgrbk(0.3))]
bad = 0
t0 = time.perf_counter()
for c in range(cases):
    kind = rng.integers(0, 4)
    if kind == 0:    # tiny
        m, p, q, n = rng.integers(2, 200), rng.integers(1, 60), rng.integers(1, 60), rng.integers(1, 300)
    elif kind == 1:  # persistent general / latency range
        m, p, q, n = rng.integers(200, 2100), rng.integers(8, 200), rng.integers(8, 200), rng.integers(100, 2500)
    elif kind == 2:  # graph path, tall
        m, p, q, n = rng.integers(3000, 9000), rng.integers(8, 96), rng.integers(8, 64), rng.integers(1200, 4000)
    else:            # graph path, wide
        m, p, q, n = rng.integers(600, 2500), rng.integers(8, 96), rng.integers(8, 64), rng.integers(8000, 16000)
    m, p, q, n = int(m), int(p), int(q), int(n)
    tag, theta, meth = meths[rng.integers(0, len(meths))]
    gram = int(rng.integers(-1, 2))
    steps = 150
    gseed = int(rng.integers(1, 10 ** 6))
    if only is not None and c not in only:
        continue
    A, B, X, Cm = O.generate(orc, gseed, m, p, q, n)
    cfg_o = O.make_config(method=tag, theta=theta, seed=7, stop_kind=O.SOLUTION_RRN, tol=0.0,
                          reference=X, refresh_interval=0)
    desc = f"case {c}: {m}x{p}.{q}x{n} {meth} cache_gram={gram}"
    try:
        so = O.Solver(orc, A, B, Cm, None, cfg_o)
        ro = so.steps(steps)
        cfg = axb.SolveConfig(method=meth, stop=axb.StopRule.solution_rrn(0.0, X), seed=7,
                              refresh_interval=0)
        sg = axb.Solver(A, B, Cm, None, cfg, axb.Options(cache_gram=gram))
        rg = sg.steps(steps)
        mism = np.nonzero(ro != rg)[0]
        e = np.linalg.norm(sg.X() - so.X()) / max(np.linalg.norm(so.X()), 1e-300)
        ok = mism.size == 0 and e <= 1e-10
        if not ok:
            bad += 1
        print(f"{'ok ' if ok else 'BAD'} {desc}: first mismatch {mism[:3]}, |dX|/|X| {e:.2e}", flush=True)
        if mism.size:
            print("    " + diagnose(orc, A, B, Cm, X, tag, theta, 7, int(mism[0])), flush=True)
    except Exception as ex:  # noqa: BLE001
        bad += 1
        print(f"ERR {desc}: {type(ex).__name__}: {ex}", flush=True)
print(f"{cases - bad}/{cases} ok in {time.perf_counter() - t0:.0f} s")
