#!/usr/bin/env python3
"""Benchmark-harness throughput: pool.benchmark on the device vs
the reference's own thread pool pattern on the host.

Workload: the acceptance-C7 style sweep — P config-1 problems (A 500×100,
B 80×400, Gaussian) × {RBK, GRBK, MWRBK} × T trials to ‖X−X*‖/‖X*‖ < 1e-6.
Device: pool.benchmark batched (run_many: one CTA per solve, one launch per
refresh segment) and threaded (`jobs` host threads, one handle and stream each).
Host: the reference engine (oracle/_ref, unmodified solver.hpp) on a bounded
sample of the same tasks, one solve per thread, all host threads.
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle_lib as O  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--problems", type=int, default=2)
    ap.add_argument("--trials", type=int, default=20)
    ap.add_argument("--jobs", default="16", help="threaded (unbatched) pool sizes to time")
    ap.add_argument("--cpu-sample", type=int, default=32, help="tasks timed on the host")
    args = ap.parse_args()
    import paper_2408_05444_b200 as P
    from paper_2408_05444_b200 import pool

    orc = O.oracle()
    probs = []
    for k in range(args.problems):
        A, B, X, Cm = O.generate(orc, 100 + k, 500, 100, 80, 400)
        probs.append(pool.BenchProblem(f"p{k}", A, B, Cm, X))
    methods = [P.Method.rbk(), P.Method.grbk(), P.Method.mwrbk()]
    ntask = len(probs) * len(methods) * args.trials
    out = {"workload": f"{len(probs)} config-1 problems x 3 methods x {args.trials} trials "
                       f"to rrn 1e-12 ({ntask} solves)", "device": {}}
    runs = [("batched", dict(batched=True, jobs=16))]
    runs += [(f"threaded_jobs{j}", dict(batched=False, jobs=int(j))) for j in args.jobs.split(",") if j]
    for label, kw in runs:
        opt = pool.BenchmarkOptions(trials=args.trials, seed=1, tol=1e-12, **kw)
        t0 = time.perf_counter()
        rows = pool.benchmark(probs, methods, opt)
        dt = time.perf_counter() - t0
        its = sum(r.it_mean * (r.trials - r.failures) for r in rows)
        out["device"][label] = {"seconds": dt, "solves_per_s": ntask / dt,
                                     "iterations_per_s": its / dt,
                                     "failures": sum(r.failures for r in rows)}
    if O.ref_available():
        ref = O.ref()
        tasks = [(p, mt, t) for p in range(len(probs)) for mt in (O.RBK, O.GRBK, O.MWRBK)
                 for t in range(args.trials)][: args.cpu_sample]
        cores = os.cpu_count() or 1
        its = [0] * len(tasks)
        nxt = [0]
        lock = threading.Lock()

        def worker():
            while True:
                with lock:
                    i = nxt[0]
                    nxt[0] += 1
                if i >= len(tasks):
                    return
                p, mt, t = tasks[i]
                pb = probs[p]
                cfg = O.make_config(method=mt, stop_kind=O.SOLUTION_RRN, tol=1e-12,
                                    reference=pb.X_star, seed=pool.substream_seed(1, t))
                rep, _, _, _ = O.Solver(ref, pb.A, pb.B, pb.C, None, cfg).run(0)
                its[i] = rep.iterations

        t0 = time.perf_counter()
        th = [threading.Thread(target=worker) for _ in range(min(cores, len(tasks)))]
        for x in th:
            x.start()
        for x in th:
            x.join()
        dt = time.perf_counter() - t0
        out["host_reference"] = {"kind": "reference", "cores": min(cores, len(tasks)),
                                 "sample": f"{len(tasks)} of the {ntask} solves",
                                 "seconds": dt, "solves_per_s": len(tasks) / dt,
                                 "iterations_per_s": sum(its) / dt}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
