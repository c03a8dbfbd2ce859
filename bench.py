#!/usr/bin/env python3
"""Benchmark: Kaczmarz iterations/s of the B200 solver (BASELINE.json metric).

Workload (default --config 5, BASELINE.json configs[4]: the large row-sharded
system, the largest that fits one GPU): ME-GRBK fp64, A 65536×8192 N(0,1/8192),
B 8192×32768 N(0,1/32768), X* 8192×8192 N(0,1), C = A·X*·B, X0 = 0, stop
solution_rrn(1e-12, X*), refresh checkpoints every 1000 iterations (the reference
default; none fall inside a default run).  --config 3 (A 8192×2048, B 2048×8192,
X0 N(0,1)) and --config 1 are the other bench workloads.  One "step" = one
Kaczmarz iteration (select → y → z/X → fused R update).  Inputs are synthetic
(seeded torch RNG on the device); R (17 GB; 537 MB at config 3) exceeds the 126 MB
L2, so no explicit flush is needed between iterations.

N > 1 (torchrun): one process per GPU and ONE system, row-sharded:
each rank owns m/N rows of A, C, R and a column slice of B; per iteration the
library issues four NCCL collectives inside its CUDA graphs (y allreduce, z
allgather, one grouped allgather of the row-norm slices and shard records,
owner-row allreduce).  Strong scaling: value = K global
iterations / max-over-ranks device time.  A is generated in 8 fixed row blocks,
so the global system is bit-identical at N = 1, 2, 4, 8.  --shard forces the
sharded code path on one GPU (1-rank communicator).

--gpus N without torchrun: bench.py re-launches itself under
torch.distributed.run with N ranks (it refuses when fewer than N GPUs are
visible); under torchrun, WORLD_SIZE must equal --gpus.

The default N=1 run (config 5) also measures configs 1-4 in the same process
and carries them under "configs" (each with its own steps, roofline,
cpu_baseline and e2e), so every BASELINE config is in the driver's BENCH line.

--impl reference: the reference's own engine on the host cores — the unmodified
axb::Solver compiled from /root/reference into oracle/_ref (kind "reference"; the
bitwise-equal C port only where _ref is absent) — one solver per core as the
reference's benchmark pool runs trials (analysis.hpp:295-313).  Config 5 does not
fit the reference's constructor on a host (G = A·Aᵀ alone is 34 GB and ~10¹⁴
FLOP), so it runs on the 1/8-per-dimension instance: "steps" / "ms_per_step"
are what actually ran there, and "value" is the config-5-equivalent rate (every
per-iteration term of the reference shrinks by exactly 64; the rule is checked
at the literal size by tools/config5_cpu_literal.py).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    2: dict(m=2000, p=500, q=400, n=2000, x0="zero", scale_a=1.0, scale_b=1.0, cpu_div=1,
            kind="svd", method="mwrbk",
            desc="config2: deterministic ME-MWRBK fp64, A 2000x500 = U.diag(s).V^T and B 400x2000 "
                 "likewise (random orthonormal U, V; s log-spaced 1..1e-2), X* N(0,1), X0=0, "
                 "C=A.X*.B"),
    1: dict(m=500, p=100, q=80, n=400, x0="zero", scale_a=1.0, scale_b=1.0, cpu_div=1,
            desc="config1: ME-GRBK fp64 A 500x100, B 80x400 iid N(0,1), X0=0"),
    3: dict(m=8192, p=2048, q=2048, n=8192, x0="randn", scale_a=1.0, scale_b=1.0, cpu_div=1,
            desc="config3: ME-GRBK(theta=1/2) fp64 A 8192x2048, B 2048x8192 iid N(0,1), "
                 "X0 N(0,1), X* N(0,1), C=A.X*.B"),
    4: dict(m=1024, p=1024, q=1024, n=1024, x0="zero", scale_a=1.0, scale_b=1.0, cpu_div=1,
            channels=3, half_band=7, blur_sigma=3.0, field_sigma=8.0, noise=1e-3,
            desc="config4: colour restoration, 3 channels of 1024x1024, A = B = banded symmetric "
                 "Toeplitz Gaussian blur (sigma 3, half-band 7), X* smooth field (Gaussian-"
                 "filtered uniform noise, sigma 8 px, [0,1]), C = A.X*.B + N(0,1e-3^2); "
                 "ME-GRBK fixed budget, one channel per GPU"),
    5: dict(m=65536, p=8192, q=8192, n=32768, x0="zero", scale_a=8192 ** -0.5,
            scale_b=32768 ** -0.5, cpu_div=8,
            desc="config5: ME-GRBK fp64 A 65536x8192 N(0,1/8192), B 8192x32768 N(0,1/32768), "
                 "X* 8192x8192 N(0,1), X0=0"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class stdout_to_stderr:
    """Route C-level stdout (fd 1) to stderr, e.g. NCCL's version banner, so the
    bench's stdout carries exactly one JSON line."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# --------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------- workload
def make_svd_system(cfg, seed):
    """Config 2 (numpy, seeded): A = U·diag(σ)·Vᵀ and B likewise with Haar
    orthonormal factors (QR of Gaussian matrices, sign-fixed) and σ log-spaced
    1..1e-2, so κ(A) = κ(B) = 100; X* N(0,1); C = A·X*·B."""
    import numpy as np

    rng = np.random.default_rng(seed)

    def orth(r, c):
        qf, rf = np.linalg.qr(rng.standard_normal((r, c)))
        return qf * np.sign(np.diag(rf))

    def built(r, c):
        k = min(r, c)
        U, V = orth(r, k), orth(c, k)
        return (U * np.logspace(0.0, -2.0, k)) @ V.T

    A = built(cfg["m"], cfg["p"])
    B = built(cfg["q"], cfg["n"])
    Xs = rng.standard_normal((cfg["p"], cfg["q"]))
    return A, B, Xs, (A @ Xs) @ B


def make_inputs_device(cfg, seed, device, world=1, rank=0, blocks=8):
    """This rank's rows of A and C (A drawn in `blocks` fixed row blocks so the
    global system does not depend on the world size) plus full B, X*, X0."""
    import torch

    dev = f"cuda:{device}"
    kw = dict(dtype=torch.float64, device=dev)
    if cfg.get("kind") == "svd":
        A, B, Xs, C = make_svd_system(cfg, seed)
        mr = cfg["m"] // world
        t = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
        out = (t(A[rank * mr:(rank + 1) * mr].copy()), t(B), t(C[rank * mr:(rank + 1) * mr].copy()),
               None, t(Xs))
        torch.cuda.synchronize(device)
        return out
    mb = cfg["m"] // blocks
    per = blocks // world
    parts = []
    for b in range(rank * per, (rank + 1) * per):
        g = torch.Generator(device=dev).manual_seed(seed * 1000 + b)
        parts.append(torch.randn(mb, cfg["p"], generator=g, **kw))
    A = torch.cat(parts) * cfg["scale_a"]
    g = torch.Generator(device=dev).manual_seed(seed * 1000 + 999)
    B = torch.randn(cfg["q"], cfg["n"], generator=g, **kw) * cfg["scale_b"]
    Xs = torch.randn(cfg["p"], cfg["q"], generator=g, **kw)
    X0 = torch.randn(cfg["p"], cfg["q"], generator=g, **kw) if cfg["x0"] == "randn" else None
    C = (A @ Xs) @ B
    torch.cuda.synchronize(device)
    return A, B, C, X0, Xs


def blur_toeplitz(nn, sigma, half_band):
    """Symmetric banded Toeplitz from a normalised 1-D Gaussian, zero boundary
    (the separable 1-D analogue of imaging.hpp:93-136; config 4)."""
    import numpy as np

    k = np.arange(-half_band, half_band + 1)
    w = np.exp(-k.astype(np.float64) ** 2 / (2.0 * sigma ** 2))
    w /= w.sum()
    T = np.zeros((nn, nn))
    for d, v in zip(k, w):
        T += np.diag(np.full(nn - abs(int(d)), v), int(d))
    return T


def make_channel(cfg, seed, c):
    """Config-4 channel c: blur A = B, smooth field X*, noisy C (host, seeded)."""
    import numpy as np

    nn = cfg["n"]
    rng = np.random.default_rng(seed * 100 + c)
    T = blur_toeplitz(nn, cfg["blur_sigma"], cfg["half_band"])
    F = blur_toeplitz(nn, cfg["field_sigma"], int(3 * cfg["field_sigma"]))
    X = F @ rng.random((nn, nn)) @ F.T
    Xs = (X - X.min()) / (X.max() - X.min())
    C = T @ Xs @ T + cfg["noise"] * rng.standard_normal((nn, nn))
    return T, T.copy(), C, Xs


def psnr(ref_planes, test_planes):
    """imaging.hpp:202-215: 10·log10(1/MSE) over all samples of all channels."""
    import numpy as np

    se = sum(float(np.sum((r - t) ** 2)) for r, t in zip(ref_planes, test_planes))
    mse = se / sum(r.size for r in ref_planes)
    return float("inf") if mse == 0.0 else 10.0 * math.log10(1.0 / mse)


class Ctx:
    """Process-level run context: ranks, device, collective plumbing."""

    def __init__(self, rank, world, local):
        self.rank, self.world, self.local = rank, world, local

    def allmax(self, x):
        if self.world == 1:
            return x
        import torch
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier(self):
        import torch
        import torch.distributed as dist

        torch.cuda.synchronize(self.local)
        if self.world > 1:
            dist.barrier()


def channels_arm(args, cfg, ctx, steps, warmup, with_cpu=True, cpu_budget_s=15.0):
    """Config 4: independent colour channels, channel c on rank c mod N (no
    collective: the channels share nothing).  A rank's channels run concurrently,
    each handle's persistent kernel on its share of the SMs; value = all
    channel-iterations ÷ the slowest rank's device time."""
    import threading

    import torch
    import torch.distributed as dist

    import paper_2408_05444_b200 as axb

    rank, world, local = ctx.rank, ctx.world, ctx.local
    mine = [c for c in range(cfg["channels"]) if c % world == rank]
    data = {c: make_channel(cfg, 4, c) for c in mine}
    if getattr(args, "csr", False):
        # the blur operators as CSR (the reference's own restoration passes SparseMatrix
        # operands, imaging.hpp:183-196): they stay sparse on the device (DESIGN §7 F1)
        import scipy.sparse as sp

        data = {c: (sp.csr_matrix(d[0]), sp.csr_matrix(d[1]), d[2], d[3]) for c, d in data.items()}
    mk = lambda: axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.residual_rel(0.0),  # noqa: E731
                                 max_iter=10 ** 9, seed=42, refresh_interval=1000)
    # ‖B‖₂ on the device: the blur's top singular gap is tiny (the reference's own
    # power iteration needs >5000 steps and throws), and no oracle needs
    # the host-order α bit for bit at n = 1024
    # (tools/config4_concurrent.py: 3 channels on one B200, 49.9k it/s one after
    # another on the whole chip, 114.8k concurrently on 49 SMs each)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    share = sms // len(mine) if len(mine) > 1 else 0
    opts = axb.Options(device=local, spectral_max_iter=200000, spectral_on_device=1, sm_share=share)
    solvers = {c: axb.Solver(d[0], d[1], d[2], None, mk(), opts) for c, d in data.items()}
    for s in solvers.values():
        s.steps(warmup)
    ctx.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    th = [threading.Thread(target=s.steps, args=(steps,)) for s in solvers.values()]
    torch.cuda.synchronize(local)
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize(local)
    wall_ms = (time.perf_counter() - t0) * 1e3
    # the span of the concurrent channels: no shorter than the longest handle's own
    # device-event loop time, and bounded by the synchronised wall clock around them
    dev_ms = max([wall_ms] + [s.last_timing()["loop_ms"] for s in solvers.values()])
    launches = sum(s.last_timing()["kernel_launches"] for s in solvers.values())
    ck = clocks.stop()
    ms = ctx.allmax(dev_ms)
    units = steps * cfg["channels"]
    value = units / (ms / 1000.0)
    # quality after the budget: PSNR against X* (imaging.hpp:202-215), ‖R‖/‖C‖
    planes = {c: (solvers[c].X(), data[c][3], solvers[c].current_residual_rel()) for c in mine}
    if world > 1:
        box = [None] * world
        dist.all_gather_object(box, planes)
        planes = {k: v for part in box for k, v in part.items()}
    order = sorted(planes)
    quality = {"psnr_db": round(psnr([planes[c][1] for c in order], [planes[c][0] for c in order]), 3),
               "residual_rel": [round(planes[c][2], 6) for c in order],
               "iterations_per_channel": warmup + steps}
    # latency-bound L2-resident working set: algorithmic bytes per iteration (touched
    # R rows, B twice, X rows of the band) over the device time, against HBM peak
    peak, peak_kind = peaks()
    hb = cfg["half_band"]
    nn = cfg["n"]
    touched = min(nn, 4 * hb + 1)
    it_bytes = 16 * touched * nn + 16 * nn * nn + 16 * (2 * hb + 1) * nn + 8 * (2 * nn)
    per_it_s = dev_ms / 1000.0 / (steps * max(1, len(mine)))
    achieved = it_bytes / per_it_s / 1e9
    # e2e: the public API from host buffers — create every channel's solver
    # (H2D, ‖B‖₂, G, R0), K steps, X back — slowest rank, wall clock
    e2e = None
    if not args.no_e2e:
        solvers = None  # release the timed handles first
        ctx.barrier()
        # the handles are created one after another (a create's device ‖B‖₂ would
        # otherwise run on the SMs the other channels' persistent kernels leave
        # free), then iterate concurrently, then X() comes back per channel
        t0 = time.perf_counter()
        hs = [axb.Solver(d[0], d[1], d[2], None, mk(), opts) for d in data.values()]
        th = [threading.Thread(target=h.steps, args=(steps,)) for h in hs]
        for t in th:
            t.start()
        for t in th:
            t.join()
        outs = [h.X() for h in hs]
        torch.cuda.synchronize(local)
        e2e_s = ctx.allmax(time.perf_counter() - t0)
        nb = lambda a: a.nbytes if hasattr(a, "nbytes") else a.data.nbytes + a.indices.nbytes + a.indptr.nbytes  # noqa: E731
        h2d = sum(nb(d[0]) + nb(d[1]) + d[2].nbytes for d in data.values())
        d2h = sum(o.nbytes for o in outs)
        e2e = {"value": units / e2e_s, "unit": "iter/s",
               "h2d_bytes_per_step": h2d // steps, "d2h_bytes_per_step": d2h // steps,
               "seconds": round(e2e_s, 4),
               "what": "Solver(host A,B,C) per channel, then steps(K) of every channel "
                       "concurrently, then X() per channel, through the C-ABI"}
        del hs
    cpu = None
    if rank == 0 and with_cpu:
        cpu = cpu_baseline(cfg, cpu_budget_s)
    return {
        "metric": "kaczmarz_iterations_per_sec", "value": round(value, 2), "unit": "iter/s",
        "n_gpus": world, "steps": steps, "warmup": warmup,
        "ms_per_step": round(ms / steps, 5), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (numpy seeded blur operator, smooth field, Gaussian noise)",
        "config": {"workload": cfg["desc"], "m": nn, "p": nn, "q": nn, "n": nn,
                   "channels": cfg["channels"], "method": "grbk", "refresh_interval": 1000,
                   "operands": "CSR" if getattr(args, "csr", False) else "dense",
                   "parallelism": f"channel c on GPU c mod {world} (independent solves, no collective; "
                                  f"a GPU's channels run concurrently on equal SM shares)",
                   "l2": "per-channel working set (40 MB) is L2-resident: latency-bound"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None, "peak_kind": peak_kind,
                     "kernel": "k_persist (persistent iteration kernel: y, z, X, banded R update, select)",
                     "algorithmic_bytes_per_iteration": it_bytes,
                     "note": "L2-resident and latency-bound; HBM fraction shown for scale only"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": ck,
        "quality": quality,
    }


def solver_config(axb, Xs, max_iter, method="grbk"):
    meth = axb.Method.mwrbk() if method == "mwrbk" else axb.Method.grbk()
    return axb.SolveConfig(method=meth, alpha_rule=axb.AlphaRule.Safe,
                           stop=axb.StopRule.solution_rrn(1e-12, Xs), max_iter=max_iter,
                           seed=42, refresh_interval=1000)


def k2_bytes(cfg, world=1):
    """Algorithmic bytes of one fused residual-update launch on one
    rank: read+write its R rows (16·m_loc·n), read the G column and z, write
    ‖R_l‖² (8·(2·m_loc + n)); m_loc = m / world."""
    m, n = cfg["m"] // world, cfg["n"]
    return 16 * m * n + 8 * (2 * m + n)


def iteration_bytes(cfg, gram_cached=True, track_ref=True, world=1):
    """Whole-iteration algorithmic bytes on one rank: K2, two passes over its
    column slice of B (y, z), its rows of X read and written, X_ref read for the
    solution_rrn error (the reference's err_sq update in update_row,
    solver.hpp:272-289; the bench's stop rule), and the G column (or its rows of A
    once more for g = A·A_iᵀ when G is not cached)."""
    m, p, q, n = cfg["m"] // world, cfg["p"], cfg["q"], cfg["n"]
    nl, pl = -(-n // world), -(-p // world)
    return (k2_bytes(cfg, world) + 16 * q * nl + 16 * pl * q + (8 * pl * q if track_ref else 0)
            + (8 * m if gram_cached else 8 * m * p))


# --------------------------------------------------------------------- CPU legs
def cpu_sample_cfg(cfg):
    """The CPU legs run the reference's per-iteration algorithm on the workload
    itself, or (config 5: its R alone is 17 GB and the reference constructor
    needs ~10¹⁴ FLOP) on the instance with every dimension divided by cpu_div.
    Each per-iteration term of the reference (R update m·n, z = BᵀB·R_iᵀ n²,
    y q·n, X p·q) then shrinks by exactly cpu_div², which scales the time back."""
    d = cfg["cpu_div"]
    c = dict(cfg)
    for k in ("m", "p", "q", "n"):
        c[k] = cfg[k] // d
    c["scale_a"] = c["p"] ** -0.5 if cfg["scale_a"] != 1.0 else 1.0
    c["scale_b"] = c["n"] ** -0.5 if cfg["scale_b"] != 1.0 else 1.0
    return c, d * d


def cpu_prepared_state(cfg, seed):
    """Host inputs + the reference constructor's caches (numpy BLAS: setup only)."""
    import numpy as np

    if "channels" in cfg:  # config 4: one blur channel (A = B = Toeplitz, X0 = 0)
        A, B, C, Xs = make_channel(cfg, 4, 0)
        X0 = np.zeros_like(Xs)
        alpha = 1.0 / float(np.linalg.eigvalsh(B @ B.T).max())
        return dict(A=A, B=B, C=C, X0=X0, Xs=Xs, R0=C.copy(), G=A @ A.T, BtB=B.T @ B, alpha=alpha)
    rng = np.random.default_rng(seed)
    m, p, q, n = cfg["m"], cfg["p"], cfg["q"], cfg["n"]
    if cfg.get("kind") == "svd":
        A, B, Xs, C = make_svd_system(cfg, seed)
    else:
        A = rng.standard_normal((m, p)) * cfg["scale_a"]
        B = rng.standard_normal((q, n)) * cfg["scale_b"]
        Xs = rng.standard_normal((p, q))
        C = (A @ Xs) @ B
    X0 = rng.standard_normal((p, q)) if cfg["x0"] == "randn" else np.zeros((p, q))
    R0 = C - (A @ X0) @ B
    G = A @ A.T
    BtB = B.T @ B
    bbt = B @ B.T if q <= n else B.T @ B
    alpha = 1.0 / float(np.linalg.eigvalsh(bbt).max())
    return dict(A=A, B=B, C=C, X0=X0, Xs=Xs, R0=R0, G=G, BtB=BtB, alpha=alpha)


def cpu_solver(O, orc, state, seed, method="grbk"):
    cfg_o = O.make_config(method=O.MWRBK if method == "mwrbk" else O.GRBK, stop_kind=O.SOLUTION_RRN, tol=1e-12,
                          reference=state["Xs"], seed=seed, refresh_interval=0)
    return O.PreparedSolver(orc, state["A"], state["B"], state["C"], state["X0"], state["R0"],
                            state["G"], state["BtB"], state["alpha"], cfg_o), cfg_o


def cpu_baseline(cfg, budget_s=15.0):
    """The oracle port (bitwise the reference's per-iteration algorithm), 1 core."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O

    orc = O.oracle()
    scfg, factor = cpu_sample_cfg(cfg)
    state = cpu_prepared_state(scfg, 7)
    s, _keep = cpu_solver(O, orc, state, 42, cfg.get("method", "grbk"))
    s.steps(1)  # warm
    t0 = time.perf_counter()
    done = 0
    while True:
        s.steps(1)
        done += 1
        if time.perf_counter() - t0 >= budget_s or done >= 2000:
            break
    dt = time.perf_counter() - t0
    shape = f"{scfg['m']}x{scfg['p']}.{scfg['q']}x{scfg['n']}"
    extra = (f"; extrapolated x{factor} to {cfg['m']}x{cfg['p']}.{cfg['q']}x{cfg['n']} "
             f"(every per-iteration term scales by {factor})" if factor > 1 else "")
    return {"value": done / dt / factor, "unit": "iter/s", "cores": 1, "kind": "port",
            "sample": f"{done} ME-{cfg.get('method', 'grbk').upper()} iterations of one {shape} solve (oracle C port of "
                      f"solver.hpp step(); constructor caches precomputed with numpy), "
                      f"{dt:.1f}s on 1 core{extra}"}


def reference_arm(args, cfg):
    """The reference's own CPU implementation of the path on the host cores: the
    UNMODIFIED reference engine (axb::Solver from /root/reference/proj/include,
    compiled with its Release flags into oracle/_ref/libaxbref.so; kind
    "reference"), one solver per host thread as the reference's benchmark pool
    runs trials (analysis.hpp:295-313).  Falls back to the bitwise-equal C port
    (kind "port") only where _ref was not built.  Config 5 runs on the exact
    1/8-per-dimension instance (its own constructor: G = A·Aᵀ, BᵀB, R0, ‖B‖₂ by
    the reference's power iteration), time extrapolated ×64."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    import oracle_lib as O

    avail = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    T = max(1, min(avail, args.ref_threads) if args.ref_threads > 0 else avail)
    # config 4: the reference constructor's spectral_norm(B) (cap 5000, tol 1e-10,
    # decomp.hpp:207-239) throws ConvergenceError for the 1024-wide blur,
    # so only the bitwise-equal port can run it
    kind = "reference" if O.ref_available() and "channels" not in cfg else "port"
    scfg, factor = cpu_sample_cfg(cfg)
    log(f"[reference] {cfg['desc']}: {kind} engine, {T} solver threads, instance "
        f"{scfg['m']}x{scfg['p']}.{scfg['q']}x{scfg['n']}")
    state = cpu_prepared_state(scfg, 7)
    solvers = [None] * T
    if kind == "reference":
        lib = O.ref()
        X0 = None if not np.any(state["X0"]) else state["X0"]

        def build(t):
            cfg_o = O.make_config(method=O.MWRBK if cfg.get("method") == "mwrbk" else O.GRBK,
                                  stop_kind=O.SOLUTION_RRN, tol=1e-12,
                                  reference=state["Xs"], seed=42 + t, refresh_interval=0)
            solvers[t] = O.Solver(lib, state["A"], state["B"], state["C"], X0, cfg_o)
    else:
        orc = O.oracle()

        def build(t):
            solvers[t] = cpu_solver(O, orc, state, 42 + t, cfg.get("method", "grbk"))[0]
    t0 = time.perf_counter()
    th = [threading.Thread(target=build, args=(t,)) for t in range(T)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    ctor_s = time.perf_counter() - t0
    log(f"[reference] {T} constructors in {ctor_s:.1f}s")
    # warmup (W iterations spread over the pool)
    wper = max(1, math.ceil(args.warmup / T))
    for s in solvers:
        s.steps(wper)
    # calibrate: bound the sample so the run stays within the budget
    t0 = time.perf_counter()
    solvers[0].steps(1)
    one = time.perf_counter() - t0
    per = max(1, math.ceil(args.steps / T))
    per = max(1, min(per, int(args.ref_budget_s / max(one, 1e-9) / 1.5)))
    per = max(per, min(int(10.0 / max(one, 1e-9)), 10 ** 6))  # at least ~10 s of CPU work
    counts = [0] * T

    def work(t):
        solvers[t].steps(per)
        counts[t] = per

    threads = [threading.Thread(target=work, args=(t,)) for t in range(T)]
    t0 = time.perf_counter()
    for x in threads:
        x.start()
    for x in threads:
        x.join()
    dt = time.perf_counter() - t0
    total = sum(counts)
    sample_rate = total / dt  # iterations/s actually run, on the instance actually run
    value = sample_rate / factor  # config-equivalent rate (== sample_rate when factor is 1)
    shape = f"{scfg['m']}x{scfg['p']}.{scfg['q']}x{scfg['n']}"
    extra = (f"; instance {shape} (every dimension /{cfg['cpu_div']}), config-{cfg['m']}x{cfg['p']}."
             f"{cfg['q']}x{cfg['n']}-equivalent rate = sample rate / {factor}" if factor > 1 else "")
    engine = ("unmodified reference axb::Solver::step() (oracle/_ref, -O3 -DNDEBUG)"
              if kind == "reference" else "oracle C port of solver.hpp step()")
    line = {
        "impl": "reference",
        "metric": "kaczmarz_iterations_per_sec", "value": value, "unit": "iter/s",
        "n_gpus": args.gpus,
        # what actually ran: `steps` iterations over the pool in steps × ms_per_step
        "steps": total, "warmup": wper * T,
        "ms_per_step": 1000.0 * dt / total,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic (numpy seeded blur operator, smooth field, noise)" if "channels" in cfg
                 else "synthetic (numpy seeded N(0,1))"),
        "config": {"workload": cfg["desc"], "m": cfg["m"], "p": cfg["p"], "q": cfg["q"],
                   "n": cfg["n"], "method": cfg.get("method", "grbk"),
                   "parallelism": f"{T} independent solves"},
        "sample": {"instance": shape, "solvers": T, "iterations": total, "seconds": round(dt, 3),
                   "iter_per_s": sample_rate, "constructors_s": round(ctor_s, 1)},
        "cpu_baseline": {"value": value, "unit": "iter/s", "cores": T, "kind": kind,
                         "sample": f"{T} concurrent solves x {per} iterations (reference "
                                   f"benchmark-pool pattern), {engine}, {dt:.1f}s wall{extra}"},
        "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if factor > 1:
        line["extrapolation"] = {
            "factor": factor, "value_is": "sample iter_per_s / factor",
            "rule": ("each per-iteration term of the reference (R update m*n, z = B^T B R_i^T n^2, "
                     "y q*n, X p*q) shrinks by exactly cpu_div^2 on the instance with every "
                     "dimension divided by cpu_div"),
            "literal_size_check": "tools/config5_cpu_literal.py (profiles/r2_config5_cpu_literal.json)"}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- GPU arm
# Sub-configurations measured in the default N=1 run, each with the number of
# timed iterations that keeps its timed region ≳ 0.1 s: config 1 (13 µs/iteration),
# config 2 (its BASELINE budget, 10⁴ MWRBK steps), config 3 (short of the first
# refresh), config 4 (3 channels concurrently).
SUB_STEPS = {1: 20000, 2: 10000, 3: 600, 4: 20000}


def system_arm(args, cfg, cfg_id, ctx, steps, warmup, sharded=False, comm=0,
               with_cpu=True, cpu_budget_s=15.0, with_tol=False):
    """One system (single GPU, or row-sharded over the ranks); returns the line."""
    import torch

    import paper_2408_05444_b200 as axb

    rank, world, local = ctx.rank, ctx.world, ctx.local
    seed = 1000
    max_iter = 10 ** 9
    if sharded:
        from paper_2408_05444_b200 import shard
    log(f"[rank {rank}] generating {cfg['desc']} (rows {rank}/{world})")
    A, B, C, X0, Xs = make_inputs_device(cfg, seed, local, world, rank)
    sopts = dict(spectral_max_iter=200000)
    meth = cfg.get("method", "grbk")

    def make_solver(A_, B_, C_, X0_, Xs_, budget=max_iter):
        if sharded:
            return shard.sharded_solver(A_, B_, C_, X0_, solver_config(axb, Xs_, budget, meth), comm,
                                        world, rank, device=local, **sopts)
        return axb.Solver(A_, B_, C_, X0_, solver_config(axb, Xs_, budget, meth),
                          axb.Options(device=local, **sopts))

    t0 = time.perf_counter()
    s = make_solver(A, B, C, X0, Xs)
    setup_s = time.perf_counter() - t0
    del A, B, C, X0
    torch.cuda.empty_cache()
    log(f"[rank {rank}] config {cfg_id}: solver ready in {setup_s:.2f}s, alpha={s.alpha():.6e}")

    # warmup, then exactly K timed steps (device events on the solver stream)
    s.steps(warmup, mirror_refresh=True)
    clocks = ClockSampler(local)
    ctx.barrier()
    clocks.start()
    ctx.barrier()
    s.steps(steps, mirror_refresh=True)
    ctx.barrier()
    ck = clocks.stop()
    tm = s.last_timing()
    ms = ctx.allmax(tm["loop_ms"])
    launches = tm["kernel_launches"]
    persistent = launches < steps  # one persistent kernel runs a whole batch
    value = steps / (ms / 1000.0)  # K global iterations of one system
    log(f"[rank {rank}] config {cfg_id}: {steps} iterations in {tm['loop_ms']:.2f} ms -> "
        f"{steps / (tm['loop_ms'] / 1000):.1f} it/s")
    per_iter_ms = ms / steps
    peak, peak_kind = peaks()
    gram = bool(s.gram_cached())
    it_bytes = iteration_bytes(cfg, gram, world=world)
    coll = None
    if persistent:
        # the dominant (only) kernel is the persistent iteration kernel: its
        # algorithmic bytes per launch over its launch time = per iteration
        achieved = it_bytes / (per_iter_ms / 1000.0) / 1e9
        roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "traffic": None, "peak_kind": peak_kind,
                    "kernel": "k_persist (one persistent cooperative kernel per batch: select, y, z/X, "
                              "fused R update + norms)",
                    "algorithmic_bytes_per_iteration": it_bytes,
                    "note": "working set L2-resident: latency-bound (grid barriers, dependent L2 "
                            "round trips); the HBM fraction is shown for scale only"}
    else:
        # dominant kernel K2 (fused residual update): CUDA events around each launch
        s.set_profiling(True)
        s.steps(args.profile_steps, mirror_refresh=False)
        pt = s.last_timing()
        kt = s.kernel_times()
        if sharded:
            coll = {k: round(v, 5) for k, v in s.collective_times().items()}
        s.set_profiling(False)
        k2_ms = pt["k2_ms"] / max(pt["k2_launches"], 1)
        kb = k2_bytes(cfg, world)
        achieved = kb / (k2_ms / 1000.0) / 1e9
        traffic, tsrc = None, None
        tf = os.path.join(ROOT, "profiles", f"k2_traffic_config{cfg_id}.json")
        if os.path.exists(tf) and world == 1:
            try:
                tj = json.load(open(tf))
                traffic, tsrc = tj.get("dram_bytes_per_launch"), tj.get("source")
            except Exception:
                traffic = None
        roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "traffic": traffic,
                    "traffic_source": tsrc or ("not measured for this shard" if world > 1 else None),
                    "kernel": "k_r_tma<true> (fused R update + row norms, TMA ring) timed together with "
                              "k_sel_greedy (next-row greedy select across the SMs)",
                    "algorithmic_bytes_per_launch": kb, "k2_ms": round(k2_ms, 5),
                    "peak_kind": peak_kind,
                    "k2_share_of_step": round(k2_ms / per_iter_ms, 4),
                    "in_pipeline_ms": {"k_yg": round(kt["yg_ms"], 5), "k_zx": round(kt["zx_ms"], 5),
                                       "k_r_tma": round(kt["k2_ms"], 5)}}
    roofline["iteration_bytes"] = it_bytes
    roofline["iteration_achieved_gbs"] = round(it_bytes / (per_iter_ms / 1000) / 1e9, 1)
    del s
    torch.cuda.empty_cache()

    # e2e: the public API from pinned host buffers (H2D of the system, device init,
    # K iterations, D2H of X), wall clock, max over ranks
    e2e = None
    if not args.no_e2e:
        Ad, Bd, Cd, X0d, Xsd = make_inputs_device(cfg, seed + 7919, local, world, rank)
        host = {}
        for name, t in (("A", Ad), ("B", Bd), ("C", Cd), ("X0", X0d), ("Xs", Xsd)):
            if t is None:
                host[name] = None
                continue
            h = torch.empty(t.shape, dtype=torch.float64, pin_memory=True)
            h.copy_(t)
            host[name] = h.numpy()
        del Ad, Bd, Cd, X0d, Xsd
        torch.cuda.empty_cache()
        h2d = sum(v.nbytes for v in host.values() if v is not None)
        # one untimed warm-up pass of the same calls (create, W steps, X()), as the
        # device-timed value has its W warm-up steps: the first create of a given
        # size in a process pays the driver's first mapping of its ~41 GB (config 5:
        # 0.9-1.2 s instead of ~0.5 s, tools/e2e_breakdown.py)
        w = make_solver(host["A"], host["B"], host["C"], host["X0"], host["Xs"], budget=steps)
        w.steps(warmup, mirror_refresh=True)
        w.X()
        del w
        ctx.barrier()
        t0 = time.perf_counter()
        # the user's budget is the K iterations it asks for (max_iter = K): the
        # solver then caches G = A·Aᵀ only if K iterations repay forming it
        s2 = make_solver(host["A"], host["B"], host["C"], host["X0"], host["Xs"], budget=steps)
        gram_e2e = bool(s2.gram_cached())
        s2.steps(steps, mirror_refresh=True)
        Xout = s2.X()
        torch.cuda.synchronize(local)
        e2e_s = ctx.allmax(time.perf_counter() - t0)
        d2h = Xout.nbytes + 8 * steps
        e2e = {"value": steps / e2e_s, "unit": "iter/s",
               "h2d_bytes_per_step": h2d // steps, "d2h_bytes_per_step": d2h // steps,
               "seconds": round(e2e_s, 4),
               "gram_cached": gram_e2e,
               "what": "Solver(host A,B,C,X0,X*, max_iter=K) -> steps(K) -> X() through the "
                       "C-ABI; includes H2D of the system, device ||B||_2, R0 (DMMA), G=A.A^T "
                       "when K repays forming it (else g=A.A_i^T per step), D2H of X; after one "
                       "untimed warm-up pass of the same calls with W steps"}
        del s2
        host = None

    # time-to-tolerance on config 1 (the reference's CPU-runnable case)
    ttt = None
    if rank == 0 and with_tol:
        try:
            ttt = time_to_tol(axb, local)
        except Exception as ex:  # noqa: BLE001  (a side measurement: keep the line)
            log(f"[bench] time_to_tol failed: {type(ex).__name__}: {ex}")
            ttt = {"error": f"{type(ex).__name__}: {ex}"}

    cpu = None
    if rank == 0 and with_cpu:
        try:
            cpu = cpu_baseline(cfg, cpu_budget_s)
        except Exception as ex:  # noqa: BLE001
            log(f"[bench] cpu_baseline failed: {type(ex).__name__}: {ex}")
            cpu = {"error": f"{type(ex).__name__}: {ex}"}
    line = {
        "metric": "kaczmarz_iterations_per_sec", "value": round(value, 2), "unit": "iter/s",
        "n_gpus": world, "steps": steps, "warmup": warmup,
        "ms_per_step": round(ms / steps, 5), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic (numpy seeded SVD-built A, B; N(0,1) X*)" if cfg.get("kind") == "svd"
                 else "synthetic (seeded torch N(0,1) on device)"),
        "config": {"workload": cfg["desc"], "m": cfg["m"], "p": cfg["p"], "q": cfg["q"],
                   "n": cfg["n"], "method": meth, "refresh_interval": 1000,
                   "gram_cached": gram,
                   "parallelism": (f"row-sharded over {world} GPUs (NCCL)" if sharded
                                   else "single GPU"),
                   "l2": ("R is 8*m*n bytes > 126 MB L2: inputs larger than L2, no flush"
                          if 8 * cfg["m"] * cfg["n"] / world > 126e6 else
                          "working set L2-resident by design (one persistent kernel per batch; "
                          "each iteration's writes are the next one's inputs): no flush")},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": ck,
        "setup_s": round(setup_s, 3),
    }
    if ttt is not None:
        line["time_to_tol"] = ttt
    if coll is not None:
        line["collectives_ms_per_iteration"] = coll
    return line


def time_to_tol(axb, local):
    """Config 1 run() to ‖X−X*‖/‖X*‖ < 1e-6 (squared RRN 1e-12)."""
    c1 = CONFIGS[1]
    A1, B1, C1, _, X1 = make_inputs_device(c1, 7, local, 1, 0, blocks=4)
    s1 = axb.Solver(A1, B1, C1, None, solver_config(axb, X1, 10 ** 6), axb.Options(device=local))
    rep = s1.run()
    out = {"config": "config1 (A 500x100, B 80x400, GRBK, ||X-X*||/||X*|| < 1e-6)",
           "iterations": rep.iterations, "seconds": round(rep.wall_seconds, 4),
           "device_loop_ms": round(s1.last_timing()["loop_ms"], 3),
           "final_rel_error": math.sqrt(rep.final_rrn),
           "terminated_by": rep.terminated_by.name}
    del s1
    return out


def self_launch(args):
    """--gpus N without a torchrun environment: re-run this command as N ranks."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        log(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible; refusing to "
            f"measure fewer GPUs than asked")
        sys.exit(2)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *sys.argv[1:]]
    log("[bench] " + " ".join(cmd))
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=5, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-tol", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="N=1 config 5: skip configs 1-4")
    ap.add_argument("--profile-steps", type=int, default=50)
    ap.add_argument("--ref-threads", type=int, default=0,
                    help="reference arm solver threads (0: every host thread this process may use)")
    ap.add_argument("--ref-budget-s", type=float, default=60.0)
    ap.add_argument("--shard", action="store_true",
                    help="use the row-sharded path even on one GPU (1-rank NCCL communicator)")
    ap.add_argument("--watchdog-s", type=float, default=1500.0)
    ap.add_argument("--csr", action="store_true",
                    help="config 4: pass the blur operators as CSR (default: dense arrays)")
    ap.add_argument("--half-band", type=int, default=None,
                    help="config 4: blur half-band (default 7; BASELINE's 'bandwidth 15' read "
                         "as half-band 7, half-band 15 the other reading, SURVEY §8 D4)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = dict(CONFIGS[args.config])
    if args.half_band is not None and "half_band" in cfg:
        cfg["desc"] = cfg["desc"].replace(f"half-band {cfg['half_band']}", f"half-band {args.half_band}")
        cfg["half_band"] = args.half_band

    in_torchrun = "WORLD_SIZE" in os.environ
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, cfg)
        return
    if not in_torchrun and args.gpus > 1:
        self_launch(args)
    if in_torchrun and world != args.gpus:
        log(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
        sys.exit(2)

    import faulthandler

    faulthandler.dump_traceback_later(args.watchdog_s, exit=True)  # never hang the box

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    ctx = Ctx(rank, world, local)

    if "channels" in cfg:
        line = channels_arm(args, cfg, ctx, args.steps, args.warmup,
                            with_cpu=not args.no_cpu_baseline)
    else:
        sharded = world > 1 or args.shard
        comm = 0
        if sharded:
            from paper_2408_05444_b200 import shard

            with stdout_to_stderr():
                if world == 1:
                    comm = shard.nccl_comm_create(1, shard.nccl_unique_id(), 0, local)
                else:
                    comm, _, _ = shard.init_comm(local)
        line = system_arm(args, cfg, args.config, ctx, args.steps, args.warmup, sharded, comm,
                          with_cpu=not args.no_cpu_baseline, with_tol=not args.no_tol)
        if sharded:
            shard.nccl_comm_destroy(comm)
    # the other BASELINE configs in the same process (N=1 default run): D1-D4
    if world == 1 and args.config == 5 and not args.no_sub and not args.shard:
        subs = {}
        for c in (1, 2, 3, 4):
            sc = dict(CONFIGS[c])
            k = SUB_STEPS[c]
            # a failing side measurement must not take the headline line with it
            try:
                if "channels" in sc:
                    subs[str(c)] = channels_arm(args, sc, ctx, k, args.warmup,
                                                with_cpu=not args.no_cpu_baseline, cpu_budget_s=10.0)
                else:
                    subs[str(c)] = system_arm(args, sc, c, ctx, k, args.warmup,
                                              with_cpu=not args.no_cpu_baseline, cpu_budget_s=10.0,
                                              with_tol=(c == 1 and not args.no_tol))
            except Exception as ex:  # noqa: BLE001
                log(f"[bench] config {c} failed: {type(ex).__name__}: {ex}")
                subs[str(c)] = {"error": f"{type(ex).__name__}: {ex}"}
            torch.cuda.empty_cache()
        line["configs"] = subs
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
