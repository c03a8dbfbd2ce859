"""Where bench.py's e2e time goes (config 5 by default): raw pinned H2D rate,
Solver(host inputs, max_iter=K) creation, K steps, X() read-back."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2408_05444_b200 as axb
from bench import CONFIGS, make_inputs_device, solver_config

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 5
K = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = CONFIGS[cfgn]
Ad, Bd, Cd, X0d, Xsd = make_inputs_device(cfg, 1000 + 7919, 0)
host = {}
for k, t in (("A", Ad), ("B", Bd), ("C", Cd), ("X0", X0d), ("Xs", Xsd)):
    if t is None:
        host[k] = None
        continue
    h = torch.empty(t.shape, dtype=torch.float64, pin_memory=True)
    h.copy_(t)
    host[k] = h
del Ad, Bd, Cd, X0d, Xsd
torch.cuda.empty_cache()
nbytes = sum(v.numel() * 8 for v in host.values() if v is not None)
dst = torch.empty_like(host["C"], device="cuda")
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dst.copy_(host["C"], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"raw pinned H2D of C ({host['C'].numel()*8/1e9:.2f} GB): {dt*1e3:.1f} ms = "
          f"{host['C'].numel()*8/dt/1e9:.1f} GB/s; whole system {nbytes/1e9:.2f} GB -> "
          f"{nbytes/(host['C'].numel()*8/dt)*1e3:.0f} ms at that rate", flush=True)
del dst
torch.cuda.empty_cache()
hn = {k: (v.numpy() if v is not None else None) for k, v in host.items()}
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s = axb.Solver(hn["A"], hn["B"], hn["C"], hn["X0"], solver_config(axb, hn["Xs"], K),
                   axb.Options(spectral_max_iter=200000))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    s.steps(K, mirror_refresh=True)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    X = s.X()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms (gram {s.gram_cached()}), {K} steps {1e3*(t2-t1):.1f} ms "
          f"(device loop {s.last_timing()['loop_ms']:.1f}), X() {1e3*(t3-t2):.1f} ms, "
          f"total {t3-t0:.3f} s -> {K/(t3-t0):.1f} it/s", flush=True)
    del s
    torch.cuda.empty_cache()
