import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import oracle_lib as O, paper_2408_05444_b200 as axb
orc = O.oracle()
A, B, X, Cm = O.generate(orc, 21, 8192, 32, 16, 64)
def mk():
    cfg_o = O.make_config(method=O.GRBK, seed=9, stop_kind=O.SOLUTION_RRN, tol=0.0, reference=X, refresh_interval=0)
    so = O.Solver(orc, A, B, Cm, None, cfg_o)
    cfg = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.solution_rrn(0.0, X), seed=9, refresh_interval=0)
    sg = axb.Solver(A, B, Cm, None, cfg)
    return so, sg
so, sg = mk()
ro = so.steps(1500); rg = sg.steps(1500)
mm = np.nonzero(ro != rg)[0]
print("mismatches", mm[:10], len(mm))
if len(mm):
    k = int(mm[0])
    so, sg = mk()
    so.steps(k); sg.steps(k)
    rs_o, rs_g = so.r_sq(), sg.residual_row_sq()
    print("k", k, "r_sq maxrel", np.max(np.abs(rs_g - rs_o) / np.maximum(rs_o, 1e-300)))
    print("rfro", so.residual_fro_sq, sg.residual_fro_sq(), (sg.residual_fro_sq()-so.residual_fro_sq)/so.residual_fro_sq)
    zo = so.greedy_threshold(0.5); zg = sg.grbk_threshold()
    print("zeta", zo, zg)
    s1 = so.greedy_index_set(0.5); s2 = np.array(sg.greedy_index_set(0.5))
    print("sets", len(s1), len(s2), np.array_equal(s1, s2), set(s1.tolist()) ^ set(s2.tolist()))
    a_sq = so.a_sq()
    for i in sorted(set(s1.tolist()) ^ set(s2.tolist())):
        print(" row", i, "r_sq_o", rs_o[i], "thr_o", zo*a_sq[i]*so.residual_fro_sq, "r_sq_g", rs_g[i], "thr_g", zg*a_sq[i]*sg.residual_fro_sq())
    print("next rows", so.step(), sg.step(), "expected", ro[k], rg[k])
