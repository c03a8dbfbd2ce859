"""Why a fuzzed case left the oracle's row sequence (shared by tools/fuzz_*.py).

Re-runs the oracle step by step up to the first differing step k and reports what
decides the selection there: how far the residual has fallen (‖R‖/‖C‖ before step
k against step 0), how far the reference's RUNNING ‖R‖² (solver.hpp:303) has
drifted from the fresh sum of its own row norms (the documented deviation,
DESIGN §4: the device sums fresh), and the gap between the two largest ratios
‖R_l‖²/‖A_l‖² (an argmax decided by rounding noise)."""
import numpy as np

import oracle_lib as O


def diagnose(orc, A, B, Cm, X, tag, theta, seed, k):
    so = O.Solver(orc, A, B, Cm, None, O.make_config(method=tag, theta=theta, seed=seed,
                  stop_kind=O.SOLUTION_RRN, tol=0.0, reference=X, refresh_interval=0))
    cn = np.linalg.norm(Cm)
    rel0 = np.sqrt(max(so.residual_fro_sq, 0.0)) / cn
    if k > 0:
        so.steps(int(k))
    run = so.residual_fro_sq
    r_sq, a_sq = so.r_sq(), so.a_sq()
    fresh = float(np.sum(r_sq))
    ratios = np.sort(np.where(a_sq > 0, r_sq / np.where(a_sq > 0, a_sq, 1.0), -np.inf))[::-1]
    gap = (ratios[0] - ratios[1]) / ratios[0] if len(ratios) > 1 and ratios[0] > 0 else float("nan")
    return (f"before step {k}: ||R||/||C|| {np.sqrt(max(run, 0.0)) / cn:.2e} (step 0: {rel0:.2e}), "
            f"reference running-vs-fresh ||R||^2 drift {abs(run - fresh) / max(fresh, 1e-300):.2e}, "
            f"top-two ratio gap {gap:.2e}, rank(A) <= {min(A.shape)}")
