"""Config 4 e2e phases (3 channels, 200 steps): create, concurrent steps and X()
per share of the SMs, and each channel's whole round trip on its own thread."""
import sys, time, threading
sys.path.insert(0, ".")
import torch
import paper_2408_05444_b200 as axb
from bench import CONFIGS, make_channel
cfg = dict(CONFIGS[4]); data = [make_channel(cfg, 4, c) for c in range(3)]
mk = lambda: axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.residual_rel(0.0), max_iter=10**9, seed=42, refresh_interval=1000)
for share in (0, 49, 0, 49):
    opts = axb.Options(spectral_max_iter=200000, spectral_on_device=1, sm_share=share)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    hs = [axb.Solver(d[0], d[1], d[2], None, mk(), opts) for d in data]
    torch.cuda.synchronize(); t1 = time.perf_counter()
    th = [threading.Thread(target=h.steps, args=(200,)) for h in hs]
    for t in th: t.start()
    for t in th: t.join()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    outs = [h.X() for h in hs]; t3 = time.perf_counter()
    print(f"share {share}: create {1e3*(t1-t0):.1f} ms, steps {1e3*(t2-t1):.1f} ms, X {1e3*(t3-t2):.1f} ms; loop_ms {[round(h.last_timing()['loop_ms'],2) for h in hs]}", flush=True)
    del hs

# every channel's whole round trip (create, steps, X) on its own thread
for share in (49, 49):
    opts = axb.Options(spectral_max_iter=200000, spectral_on_device=1, sm_share=share)
    outs = [None] * 3

    def one(i, d):
        h = axb.Solver(d[0], d[1], d[2], None, mk(), opts)
        h.steps(200)
        outs[i] = h.X()
        del h

    torch.cuda.synchronize(); t0 = time.perf_counter()
    th = [threading.Thread(target=one, args=(i, d)) for i, d in enumerate(data)]
    for t in th: t.start()
    for t in th: t.join()
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"share {share}, per-channel threads: total {1e3*(t1-t0):.1f} ms", flush=True)
