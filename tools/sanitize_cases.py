"""Small solves on every execution path, one per --case, for compute-sanitizer.

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck \
        python tools/sanitize_cases.py --case NAME

Cases (each a few iterations at a size the sanitizers finish in seconds):
  lat        persistent latency body (m ≤ 2048, BᵀB cached), GRBK
  general    persistent general body (AXB_PERSIST_LAT=0), RGRBK
  graph_tma  CUDA-graph path with the TMA K2 ring (AXB_PERSIST=0, even n), GRBK + k_sel_greedy
  graph_reg  CUDA-graph path with the register K2 (odd n), MWRBK
  batch      k_persist_batch: several independent solves through run_many
  sharded    the row-sharded path, 2 emulated ranks (grouped allgather, k_sel1, k_pack)
  sparse     CSR A and B (host Gram, scattered Gram row) on both persistent bodies
  analysis   F2: device Jacobi SVD / reference_solution
  checkpoint DMMA K1 residual GEMM with the fused epilogue (checkpoint, exact metrics)
Prints "<case> ok" on success.
"""
import argparse
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402


def gen(m, p, q, n, seed=3):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, p))
    B = rng.standard_normal((q, n))
    X = rng.standard_normal((p, q))
    return A, B, X, (A @ X) @ B


def cfg(axb, X, meth, k=0):
    return axb.SolveConfig(method=meth, stop=axb.StopRule.solution_rrn(0.0, X), seed=5,
                           refresh_interval=0, max_iter=10 ** 6)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", required=True)
    a = ap.parse_args()
    c = a.case
    if c == "general":
        os.environ["AXB_PERSIST_LAT"] = "0"
    if c.startswith("graph"):
        os.environ["AXB_PERSIST"] = "0"
    import paper_2408_05444_b200 as axb

    if c == "lat":
        A, B, X, Cm = gen(120, 30, 20, 90)
        s = axb.Solver(A, B, Cm, None, cfg(axb, X, axb.Method.grbk()))
        s.steps(40)
        s.X()
    elif c == "general":
        A, B, X, Cm = gen(300, 40, 24, 100)
        s = axb.Solver(A, B, Cm, None, cfg(axb, X, axb.Method.rgrbk(0.3)))
        s.steps(30)
        s.X()
    elif c == "graph_tma":
        A, B, X, Cm = gen(4096, 32, 16, 2048)  # greedy over ≥ 64 groups: k_sel_greedy
        s = axb.Solver(A, B, Cm, None, cfg(axb, X, axb.Method.grbk()))
        s.steps(6)
        s.X()
    elif c == "graph_reg":
        A, B, X, Cm = gen(256, 24, 16, 301)  # odd n: register K2
        s = axb.Solver(A, B, Cm, None, cfg(axb, X, axb.Method.mwrbk()))
        s.steps(6)
        s.X()
    elif c == "batch":
        sol = []
        for t in range(4):
            A, B, X, Cm = gen(80, 20, 12, 60, seed=t)
            sol.append(axb.Solver(A, B, Cm, None, axb.SolveConfig(
                method=axb.Method.grbk(), stop=axb.StopRule.solution_rrn(1e-8, X), seed=t,
                refresh_interval=50, max_iter=200)))
        axb.run_many(sol)
    elif c == "sharded":
        from paper_2408_05444_b200 import shard

        A, B, X, Cm = gen(128, 24, 16, 64)
        comms = shard.emulated_comms(2)
        errs = []

        def rank(r):
            try:
                sl = slice(r * 64, (r + 1) * 64)
                s = shard.sharded_solver(np.ascontiguousarray(A[sl]), B,
                                         np.ascontiguousarray(Cm[sl]), None,
                                         cfg(axb, X, axb.Method.grbk()), comms[r], 2, r)
                s.steps(8)
                s.X()
            except Exception as e:  # noqa: BLE001
                errs.append(e)

        th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for cm in comms:
            shard.nccl_comm_destroy(cm)
        if errs:
            raise errs[0]
    elif c == "sparse":
        import scipy.sparse as sp

        rng = np.random.default_rng(1)
        Ad = np.zeros((200, 150))
        for i in range(200):
            j0 = int(i * 150 / 200)
            Ad[i, max(0, j0 - 2):j0 + 3] = 1.0 + rng.random(len(range(max(0, j0 - 2), min(150, j0 + 3))))
        Bd = np.zeros((20, 60))
        for i in range(20):
            Bd[i, 3 * i:3 * i + 5] = 1.0 + rng.random(len(range(3 * i, min(60, 3 * i + 5))))
        X = rng.standard_normal((150, 20))
        Cm = (Ad @ X) @ Bd
        for lat in ("256", "0"):
            os.environ["AXB_PERSIST_LAT"] = lat
            s = axb.Solver(sp.csr_matrix(Ad), sp.csr_matrix(Bd), Cm, None, cfg(axb, X, axb.Method.grbk()))
            s.steps(20)
            s.update_row(3)
            s.checkpoint()
            s.X()
            del s
    elif c == "analysis":
        from paper_2408_05444_b200 import analysis

        A, B, X, Cm = gen(40, 12, 10, 30)
        analysis.reference_solution(A, B, Cm)
    elif c == "checkpoint":
        A, B, X, Cm = gen(300, 40, 24, 100)
        X0 = np.random.default_rng(9).standard_normal((40, 24))
        s = axb.Solver(A, B, Cm, X0, cfg(axb, X, axb.Method.grbk()))
        s.steps(10)
        s.checkpoint()
        s.exact_metric()
        s.exact_residual_rel()
    else:
        raise SystemExit(f"unknown case {c}")
    print(f"{c} ok", flush=True)


if __name__ == "__main__":
    main()
