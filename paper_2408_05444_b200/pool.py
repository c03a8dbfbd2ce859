"""Benchmark pool over the B200 path — the reference harness, device-side.

Mirrors axb::benchmark (analysis.hpp:255-356): every (problem, method, trial)
combination runs with the shared per-trial substream seed
RngStream(seed).substream(trial).seed() (:279, rng.hpp:102-104), X0 = 0; IT and
wall time are averaged over converged trials, divergent or budget-exhausted
trials are counted as failures, and each row reports its speed-up against the
RBK row of the same problem (:315-354).

Where the reference runs one solve per CPU thread, the device path batches
(SURVEY §8(f) F3): per device, the task handles are created by ``jobs`` host
threads and then advanced together by ``run_many`` (axb_solvers_run) — every
small system is one CTA of a single persistent launch per refresh segment, so
hundreds of latency-bound trials share the GPU instead of queueing.  With
``batched=False`` each of ``jobs`` threads drives its own handle's run()
(one stream each).  The C-ABI releases the GIL for the duration of each call.
"""
from __future__ import annotations

import math
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from .analysis import reference_solution
from .errors import ConfigError, DivergenceError
from .solver import (AlphaRule, Method, MethodTag, Options, SolveConfig, Solver, StopRule,
                     Terminated, run_many)

_M64 = (1 << 64) - 1


def _mix_pure(z: int) -> int:  # rng.hpp:113-117
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def substream_seed(seed: int, trial: int) -> int:
    """RngStream(seed).substream(trial).seed() — rng.hpp:102-104."""
    return (seed ^ _mix_pure((0x5851F42D4C957F2D + trial) & _M64)) & _M64


@dataclass
class BenchProblem:
    id: str
    A: np.ndarray
    B: np.ndarray
    C: np.ndarray
    X_star: Optional[np.ndarray] = None  # solution_rrn reference; None → device reference_solution


@dataclass
class BenchmarkOptions:  # analysis.hpp BenchmarkOptions
    trials: int = 20
    alpha_rule: AlphaRule = AlphaRule.Safe
    alpha_value: float = 0.0
    max_iter: int = 1000000   # analysis.hpp:220
    seed: int = 1             # analysis.hpp:221
    stop_kind: StopRule.Kind = StopRule.Kind.SolutionRrn
    tol: float = 1e-6
    jobs: int = 4
    devices: Sequence[int] = (0,)
    options: dict = field(default_factory=dict)  # extra solver Options fields
    batched: bool = True      # run_many per device (one CTA per small system)
    batch_size: int = 1184    # handles per run_many call (bounds device memory)


@dataclass
class BenchmarkRow:  # analysis.hpp:225-236
    problem_id: str
    method: str
    theta: Optional[float]
    alpha_rule: str
    trials: int
    it_mean: float = 0.0
    it_std: float = 0.0
    wall_mean_s: float = 0.0
    speed_up_vs_rbk: Optional[float] = None
    failures: int = 0


def benchmark(problems: List[BenchProblem], methods: List[Method],
              opt: BenchmarkOptions) -> List[BenchmarkRow]:
    if opt.trials < 1:
        raise ConfigError("benchmark: trials must be >= 1")
    for m in methods:
        m.validate()
    # per-problem references, as the reference harness computes them up front
    # (analysis.hpp:261-264) — on the device here
    references = []
    for i, pb in enumerate(problems):
        if pb.X_star is not None:
            references.append(pb.X_star)
        else:
            dev = opt.devices[i % len(opt.devices)]
            references.append(reference_solution(pb.A, pb.B, pb.C, device=dev).X_star)
    tasks = [(p, mi, t) for p in range(len(problems)) for mi in range(len(methods))
             for t in range(opt.trials)]
    outcomes = [None] * len(tasks)

    def make_task(idx):
        p, mi, t = tasks[idx]
        pb = problems[p]
        if opt.stop_kind == StopRule.Kind.SolutionRrn:
            stop = StopRule.solution_rrn(opt.tol, references[p])
        else:
            stop = StopRule.residual_rel(opt.tol)
        cfg = SolveConfig(method=methods[mi], alpha_rule=opt.alpha_rule,
                          alpha_value=opt.alpha_value, stop=stop, max_iter=opt.max_iter,
                          seed=substream_seed(opt.seed, t))
        dev = opt.devices[idx % len(opt.devices)]
        return Solver(pb.A, pb.B, pb.C, None, cfg, Options(device=dev, **opt.options))

    def run_task(idx):
        try:
            rep = make_task(idx).run()
            outcomes[idx] = (float(rep.iterations), rep.wall_seconds,
                             rep.terminated_by == Terminated.MaxIter)
        except DivergenceError:
            outcomes[idx] = (0.0, 0.0, True)

    jobs = max(1, min(opt.jobs, len(tasks)))

    def pool_map(fn, items):
        """fn over items on `jobs` host threads; first error re-raised."""
        nxt = [0]
        lock = threading.Lock()
        errors = []

        def worker():
            while True:
                with lock:
                    i = nxt[0]
                    nxt[0] += 1
                if i >= len(items):
                    return
                try:
                    fn(items[i])
                except Exception as e:  # surface after the pool drains
                    errors.append(e)
                    return

        threads = [threading.Thread(target=worker) for _ in range(min(jobs, len(items)))]
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        if errors:
            raise errors[0]

    if opt.batched:
        for d, dev in enumerate(opt.devices):
            mine = [i for i in range(len(tasks)) if i % len(opt.devices) == d]
            for c0 in range(0, len(mine), max(1, opt.batch_size)):
                chunk = mine[c0:c0 + max(1, opt.batch_size)]
                handles = [None] * len(chunk)

                def build(j):
                    handles[j] = make_task(chunk[j])

                pool_map(build, list(range(len(chunk))))
                results = run_many(handles, return_exceptions=True)
                for idx, res in zip(chunk, results):
                    if isinstance(res, DivergenceError):
                        outcomes[idx] = (0.0, 0.0, True)
                    elif isinstance(res, Exception):
                        raise res
                    else:
                        outcomes[idx] = (float(res.iterations), res.wall_seconds,
                                         res.terminated_by == Terminated.MaxIter)
                del handles
    else:
        pool_map(run_task, list(range(len(tasks))))

    rows, rbk_wall = [], [-1.0] * len(problems)
    for p, pb in enumerate(problems):
        for mi, m in enumerate(methods):
            row = BenchmarkRow(pb.id, m.label(), m.theta, opt.alpha_rule.name.lower(), opt.trials)
            its, walls = [], []
            for t in range(opt.trials):
                it, wall, failed = outcomes[(p * len(methods) + mi) * opt.trials + t]
                if failed:
                    row.failures += 1
                    continue
                its.append(it)
                walls.append(wall)
            if its:
                row.it_mean = sum(its) / len(its)
                row.wall_mean_s = sum(walls) / len(walls)
                var = sum((v - row.it_mean) ** 2 for v in its)
                row.it_std = math.sqrt(var / (len(its) - 1)) if len(its) > 1 else 0.0
            if m.tag == MethodTag.RBK and its:
                rbk_wall[p] = row.wall_mean_s
            rows.append(row)
    for row in rows:
        for p, pb in enumerate(problems):
            if pb.id == row.problem_id and rbk_wall[p] > 0.0 and row.wall_mean_s > 0.0:
                row.speed_up_vs_rbk = rbk_wall[p] / row.wall_mean_s
    return rows
