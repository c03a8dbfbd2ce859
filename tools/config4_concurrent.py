"""Config 4's three independent channels on ONE GPU: one after another on the whole
chip (bench.py's N=1 schedule) vs concurrently, each channel's persistent grid
limited to a share of the SMs (AXB_PERSIST_GRID) and driven from its own host
thread / stream.  Wall clock between device synchronisations.

    python tools/config4_concurrent.py [K] [grid ...]
"""
import os, sys, threading, time
sys.path.insert(0, ".")
import torch

K = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
grids = [int(g) for g in sys.argv[2:]] or [148, 74, 49]
from bench import CONFIGS, make_channel  # noqa: E402
import paper_2408_05444_b200 as axb  # noqa: E402

cfg = CONFIGS[4]
data = [make_channel(cfg, 4, c) for c in range(3)]
for grid in grids:
    os.environ["AXB_PERSIST_GRID"] = str(grid)
    mk = lambda: axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.residual_rel(0.0),  # noqa: E731
                                 max_iter=10 ** 9, seed=42, refresh_interval=1000)
    opts = axb.Options(spectral_max_iter=200000, spectral_on_device=1)
    ss = [axb.Solver(d[0], d[1], d[2], None, mk(), opts) for d in data]
    for s in ss:
        s.steps(50)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in ss:
        s.steps(K)
    torch.cuda.synchronize()
    seq = time.perf_counter() - t0
    th = [threading.Thread(target=s.steps, args=(K,)) for s in ss]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    conc = time.perf_counter() - t0
    print(f"grid {grid}: sequential {3 * K / seq:.0f} it/s, concurrent {3 * K / conc:.0f} it/s", flush=True)
    del ss
