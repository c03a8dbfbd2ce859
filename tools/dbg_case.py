"""Debug one fuzz case: oracle vs single-GPU vs emulated sharded rows."""
import sys, threading
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import oracle_lib as O
import paper_2408_05444_b200 as axb
from paper_2408_05444_b200 import shard
rng = np.random.default_rng(3)
orc = O.oracle()
for c in range(3):
    world = int(rng.choice([2, 4, 8])); ml = int(rng.integers(1, 900))
    m, p, q, n = ml * world, int(rng.integers(1, 120)), int(rng.integers(1, 90)), int(rng.integers(2, 3000))
    mi = rng.integers(0, 5); gram = int(rng.integers(0, 2)); seed = int(rng.integers(1, 10 ** 6))
print(world, m, p, q, n, mi, gram, seed)
A, B, X, Cm = O.generate(orc, seed, m, p, q, n)
so = O.Solver(orc, A, B, Cm, None, O.make_config(method=O.MWRBK, seed=9, stop_kind=O.SOLUTION_RRN,
              tol=0.0, reference=X, refresh_interval=0))
ro = []
rel = []
for k in range(120):
    ro.append(int(so.steps(1)[0]))
    rel.append(np.sqrt(max(so.residual_fro_sq, 0)) / np.linalg.norm(Cm))
ro = np.array(ro)
cfg = lambda: axb.SolveConfig(method=axb.Method.mwrbk(), stop=axb.StopRule.solution_rrn(0.0, X), seed=9, refresh_interval=0)
s1 = axb.Solver(A, B, Cm, None, cfg(), axb.Options(cache_gram=gram))
r1 = s1.steps(120)
print("single GPU first mismatch", np.nonzero(r1 != ro)[0][:5])
comms = shard.emulated_comms(world); out = [None] * world
def body(r):
    s = shard.sharded_solver(np.ascontiguousarray(A[r*ml:(r+1)*ml]), B, np.ascontiguousarray(Cm[r*ml:(r+1)*ml]),
                             None, cfg(), comms[r], world, r, cache_gram=gram)
    out[r] = s.steps(120)
th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
[t.start() for t in th]; [t.join() for t in th]
mm = np.nonzero(out[0] != ro)[0]
print("sharded first mismatch", mm[:5])
if mm.size:
    k = mm[0]
    print("at step", k, "oracle row", ro[k], "sharded row", out[0][k], "oracle ||R||/||C|| before", rel[k-1] if k else None)
