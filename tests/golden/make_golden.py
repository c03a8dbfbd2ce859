#!/usr/bin/env python3
"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libaxbref.so).

Run in the build container, where /root/reference exists and `make -C oracle`
built the reference driver.  The fixtures pin the C restatement (oracle/) and
travel with the repo; nothing here is needed at test time.

Fixtures (all produced by the reference's own code paths):
  rng.npz        xoshiro256** u64 stream and Box–Muller gauss stream for seeds
                 0, 42, 2**64-1 (rng.hpp:30-59); substream seeds (rng.hpp:102-104)
  gen_c1.npz     generate() for config 1 (seed 7): sha256 of A, B, X*, C bytes
  run_c1_*.npz   config-1 run() to ‖X−X*‖/‖X*‖ < 1e-6 (squared RRN 1e-12) for
                 GRBK / RGRBK(0.25) / MWRBK / RBK / BK, solver seed 42, refresh 1000:
                 iterations, α, final RRN, the run() trace's selected rows, final X
  kat_small.npz  test_solver.cpp-style small systems: 30-step row sequences and X
  analysis.npz   decomp.hpp svd / pseudoinverse and analysis.hpp reference_solution /
                 bk_limit on the shapes test_decomp.cpp / test_analysis.cpp use
                 (inputs from numpy default_rng, stored with the outputs)
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_lib as O  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def main():
    assert O.ref_available(), "build oracle/_ref first (make -C oracle)"
    ref = O.ref()
    # -- rng streams
    seeds = np.array([0, 42, 2**64 - 1], dtype=np.uint64)
    u64 = np.zeros((3, 256), dtype=np.uint64)
    gs = np.zeros((3, 256))
    for i, sd in enumerate(seeds):
        ref.rng_stream(int(sd), 256, u64[i].ctypes.data_as(O._u64p), O._ptr(gs[i]))
    subs = np.array([[ref.substream_seed(int(sd), t) for t in range(4)] for sd in seeds],
                    dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), seeds=seeds, u64=u64, gauss=gs,
                        substream_seeds=subs)
    # -- config-1 inputs
    A, B, X, C = O.generate(ref, 7, 500, 100, 80, 400)
    np.savez_compressed(os.path.join(HERE, "gen_c1.npz"), seed=7,
                        shape=np.array([500, 100, 80, 400]),
                        sha_A=sha(A), sha_B=sha(B), sha_X=sha(X), sha_C=sha(C),
                        A00=A[:2, :4], C00=C[:2, :4])
    # -- config-1 runs
    for name, tag, theta in [("grbk", O.GRBK, None), ("rgrbk025", O.RGRBK, 0.25),
                             ("mwrbk", O.MWRBK, None), ("rbk", O.RBK, None), ("bk", O.BK, None)]:
        cfg = O.make_config(method=tag, theta=theta, stop_kind=O.SOLUTION_RRN, tol=1e-12,
                            reference=X, seed=42, record_trace=True, max_iter=40000,
                            refresh_interval=1000)
        s = O.Solver(ref, A, B, C, None, cfg)
        rep, rows, rrn, Xf = s.run(40000)
        np.savez_compressed(os.path.join(HERE, f"run_c1_{name}.npz"), iterations=rep.iterations,
                            alpha=rep.alpha, final_rrn=rep.final_rrn,
                            final_residual_rel=rep.final_residual_rel,
                            rows=rows.astype(np.uint16), rrn=rrn[::50], X=Xf)
        print(name, rep.iterations, rep.final_rrn)
    # -- small systems, 30 steps each (NaiveRunner-style, test_solver.cpp:421-515)
    out = {}
    for k, (m, p, q, n, seed) in enumerate([(7, 4, 3, 6, 6701), (12, 5, 4, 9, 6001),
                                            (60, 20, 15, 40, 111)]):
        A2, B2, X2, C2 = O.generate(ref, seed, m, p, q, n)
        for name, tag, theta in [("bk", O.BK, None), ("grbk", O.GRBK, None),
                                 ("mwrbk", O.MWRBK, None), ("rgrbk08", O.RGRBK, 0.8),
                                 ("rbk", O.RBK, None)]:
            cfg = O.make_config(method=tag, theta=theta, alpha_rule=O.SAFE,
                                stop_kind=O.RESIDUAL_REL, tol=0.0, seed=77, refresh_interval=0)
            s = O.Solver(ref, A2, B2, C2, None, cfg)
            rows = s.steps(30)
            out[f"s{k}_{name}_rows"] = rows.astype(np.uint16)
            out[f"s{k}_{name}_X"] = s.X()
            out[f"s{k}_{name}_alpha"] = s.alpha
        out[f"s{k}_shape"] = np.array([m, p, q, n, seed])
    np.savez_compressed(os.path.join(HERE, "kat_small.npz"), **out)
    analysis_fixtures(ref)


def analysis_cases(seed=2408):
    """Inputs for analysis.npz: (name, A, B, C, X0, rank_tol)."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal

    def stacked(rows, cols):  # stack_rows_twice (test_analysis.cpp:12-20): rank `rows`
        h = g((rows, cols))
        return np.vstack([h, h])

    cases = []
    I4 = np.eye(4)
    cases.append(("identity", I4, I4, g((4, 4)), np.zeros((4, 4)), -1.0))
    for name, A, B in [("unique", g((6, 3)), g((3, 6))),            # kind 0
                       ("rowcol", g((3, 7)), g((8, 4))),            # kind 1
                       ("general", stacked(2, 5), g((4, 6))),       # kind 2
                       ("medium", g((48, 32)), g((24, 40))),        # kind 0
                       ("medium_def", stacked(10, 24), g((16, 30)))]:  # kind 2
        X = g((A.shape[1], B.shape[0]))
        cases.append((name, A, B, A @ X @ B, g(X.shape), -1.0))
    A = stacked(2, 5)
    B = g((4, 6))
    cases.append(("general_tol", A, B, A @ g((5, 4)) @ B, g((5, 4)), 1e-6))
    cases.append(("inconsistent", stacked(2, 4), g((3, 5)), g((4, 5)), np.zeros((4, 3)), -1.0))
    return cases


def svd_cases(seed=2409):
    rng = np.random.default_rng(seed)
    out = [("diag", np.array([[2.0, 0.0], [0.0, 0.0]]))]
    for r, c in [(8, 5), (5, 8), (7, 7), (12, 4), (33, 20)]:
        out.append((f"u{r}x{c}", rng.uniform(-1.0, 1.0, (r, c))))
    h = rng.uniform(-1.0, 1.0, (9, 3))
    out.append(("dupcols", np.hstack([h, h])))  # rank 3 (test_decomp.cpp:59-69)
    return out


def analysis_fixtures(ref):
    an = O.Analysis(ref)
    out = {}
    for name, M in svd_cases():
        U, s, V, rank = an.svd(M)
        out.update({f"svd_{name}_M": M, f"svd_{name}_U": U, f"svd_{name}_s": s,
                    f"svd_{name}_V": V, f"svd_{name}_rank": rank,
                    f"svd_{name}_pinv": an.pseudoinverse(M)})
    for name, A, B, Cm, X0, tol in analysis_cases():
        out.update({f"rs_{name}_A": A, f"rs_{name}_B": B, f"rs_{name}_C": Cm,
                    f"rs_{name}_X0": X0, f"rs_{name}_tol": tol})
        try:
            X, kind, res = an.reference_solution(A, B, Cm, tol)
            out.update({f"rs_{name}_X": X, f"rs_{name}_kind": kind, f"rs_{name}_res": res,
                        f"rs_{name}_code": 0})
        except O.OracleError as e:
            out.update({f"rs_{name}_code": e.code, f"rs_{name}_msg": str(e)})
        try:
            out[f"rs_{name}_bk"] = an.bk_limit(A, B, Cm, X0)
        except O.OracleError:
            pass
    out["names"] = np.array([c[0] for c in analysis_cases()])
    out["svd_names"] = np.array([c[0] for c in svd_cases()])
    np.savez_compressed(os.path.join(HERE, "analysis.npz"), **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["analysis"]:
        analysis_fixtures(O.ref())
    else:
        main()
