"""Per-rank kernel profile of the row-sharded config-5 system at world W on ONE
GPU (profiling tool; run under `ncu --metrics gpu__time_duration.sum`).

Every rank is a host thread with its own handle on cuda:0 and the library's
in-process collective emulation (axb_nccl_emulated_group), so each rank runs its
production kernels at the world-W shapes (m/W rows of R, column slices of B for
y and z, a row slice of X) and no kernel waits on another.  Wall times here are
meaningless (the ranks share one GPU); the ncu launch list gives the per-rank
kernel durations of an N = W run without its NCCL latency.

usage: python tools/emulated_shard_profile.py [W] [steps]
"""
import sys
import threading

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2408_05444_b200 as axb  # noqa: E402
from paper_2408_05444_b200 import shard  # noqa: E402
from bench import CONFIGS, make_inputs_device, solver_config  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = CONFIGS[5]
host = []
for r in range(W):  # one rank's inputs at a time on the device, then parked on the host
    A, B, C, X0, Xs = make_inputs_device(cfg, 1000, 0, W, r)
    host.append(tuple(t.cpu().numpy() if t is not None else None for t in (A, B, C, X0, Xs)))
    del A, B, C, X0, Xs
    torch.cuda.empty_cache()
comms = shard.emulated_comms(W)
solvers = [None] * W
errs = []


def body(r, fn):
    try:
        fn(r)
    except Exception as e:  # noqa: BLE001
        errs.append(e)


def run(fn):
    th = [threading.Thread(target=body, args=(r, fn)) for r in range(W)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]


def create(r):
    A, B, C, X0, Xs = host[r]
    solvers[r] = shard.sharded_solver(A, B, C, X0, solver_config(axb, Xs, 10 ** 9), comms[r], W, r,
                                      device=0, spectral_max_iter=200000, cache_gram=1)


run(create)
run(lambda r: solvers[r].steps(5, mirror_refresh=True))
run(lambda r: solvers[r].steps(steps, mirror_refresh=True))
print(f"world {W}: {steps} steps per rank done; gram cached {solvers[0].gram_cached()}", flush=True)
