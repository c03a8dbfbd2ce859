"""BASELINE config 3 at full size, the rest of its family run to tolerance on the device:
relaxed ME-GRBK at theta = 0.25 and 0.75 (full rank, X0 N(0,1)) and the rank-deficient
variant (rank(A) = 1536 by zeroing A's 512 smallest singular values), which must converge
to X0_* = A⁺CB⁺ + X0 − A⁺AX0BB⁺ (analysis.hpp:95-104), not to X*.

Each run goes through run() with the reference's default refresh every 1000 steps and
stops at ‖X − X_target‖_F/‖X_target‖_F < 1e-6 (solution_rrn 1e-12).  The rank-deficient
target is formed two ways: from the generating SVD (B has full row rank, so
BB⁺ = I and X0_* = X0 + V_r V_rᵀ (X* − X0)), and with the library's own device
bk_limit; both are reported.

    python tools/ttt_config3_family.py [--only theta0.25,theta0.75,rankdef]
"""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2408_05444_b200 as axb
from bench import CONFIGS, make_inputs_device


def run(A, B, C, X0, target, method, label, extra):
    cfg = axb.SolveConfig(method=method, alpha_rule=axb.AlphaRule.Safe,
                          stop=axb.StopRule.solution_rrn(1e-12, target), max_iter=3 * 10 ** 6,
                          seed=42, refresh_interval=1000)
    t0 = time.perf_counter()
    s = axb.Solver(A, B, C, X0, cfg, axb.Options(spectral_max_iter=200000))
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    rep = s.run()
    X = torch.from_numpy(np.ascontiguousarray(rep.X)).cuda()
    rel = float(torch.linalg.norm(X - target) / torch.linalg.norm(target))
    out = {"run": label, "method": method.tag.name + (f"({method.theta})" if method.theta else ""),
           "iterations": rep.iterations, "loop_seconds": round(rep.wall_seconds, 3),
           "setup_seconds": round(setup, 3), "terminated_by": rep.terminated_by.name,
           "final_rel_error_reported": rep.final_rrn ** 0.5, "final_rel_error_recomputed": rel,
           "us_per_iteration": round(rep.wall_seconds / max(rep.iterations, 1) * 1e6, 2),
           "alpha": s.alpha(), **extra}
    print(json.dumps(out), flush=True)
    del s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="theta0.25,theta0.75,rankdef")
    args = ap.parse_args()
    todo = args.only.split(",")
    cfg = CONFIGS[3]
    A, B, C, X0, Xs = make_inputs_device(cfg, 1000, 0)
    for th in (0.25, 0.75):
        if f"theta{th}" in todo:
            run(A, B, C, X0, Xs, axb.Method.rgrbk(th), f"config3 full rank, RGRBK theta={th}",
                {"target": "X* (A full column rank, B full row rank: X0_* = X*)"})
    if "rankdef" in todo:
        rank = 1536
        U, S, Vh = torch.linalg.svd(A, full_matrices=False)
        S[rank:] = 0.0
        Ad = (U * S) @ Vh
        Cd = (Ad @ Xs) @ B
        Vr = Vh[:rank].T
        target = X0 + Vr @ (Vr.T @ (Xs - X0))
        t0 = time.perf_counter()
        lim = torch.from_numpy(axb.analysis.bk_limit(Ad.cpu().numpy(), B.cpu().numpy(),
                                                     Cd.cpu().numpy(), X0.cpu().numpy())).cuda()
        t_lim = time.perf_counter() - t0
        d = float(torch.linalg.norm(lim - target) / torch.linalg.norm(target))
        dxs = float(torch.linalg.norm(Xs - target) / torch.linalg.norm(target))
        del U, Vh, Vr
        run(Ad, B, Cd, X0, target, axb.Method.grbk(), "config3 rank(A)=1536, GRBK",
            {"target": "X0 + V_r V_r^T (X* - X0) from the generating SVD",
             "device_bk_limit_rel_diff": d, "device_bk_limit_seconds": round(t_lim, 2),
             "x_star_rel_distance_from_target": dxs,
             "sigma_kept_min": float(S[rank - 1])})


if __name__ == "__main__":
    main()
