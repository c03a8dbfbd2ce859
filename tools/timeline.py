"""In-pipeline timeline of the graph path's iteration kernels (device clock).

Needs the library built with -DAXB_TRACE_TIMELINE (tools/timeline.sh rebuilds a
box-local copy).  Prints, per kernel, the mean span (earliest CTA start after its
dependency wait → latest CTA end) and the mean gap to the next kernel's start over
the last iterations of a run — what CUDA events cannot show, because events
serialise the programmatic-dependent-launch overlap.

  python tools/timeline.py 3        # config 3
"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2408_05444_b200 as axb
from paper_2408_05444_b200 import _lib
from bench import CONFIGS, make_inputs_device, solver_config

lib = _lib.load()
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = CONFIGS[cfg_id]
A, B, Cm, X0, Xs = make_inputs_device(cfg, 1000, 0)
s = axb.Solver(A, B, Cm, X0, solver_config(axb, Xs, 10 ** 9), axb.Options(spectral_max_iter=200000))
del A, B, Cm
s.steps(64)
buf = (C.c_uint64 * 512)()
assert lib.axb_debug_timeline(buf, 1) == 1, "library not built with -DAXB_TRACE_TIMELINE"
s.steps(64)
k_end = s.iteration()
lib.axb_debug_timeline(buf, 0)
t = np.frombuffer(buf, dtype=np.uint64).reshape(64, 4, 2).astype(np.int64)
# order the ring by iteration: slot = k & 63 for the 64 iterations before k_end
order = [(k & 63) for k in range(k_end - 64, k_end)]
t = t[order]
names = ["K4 k_yg", "K4b+K5 k_zx", "K2 k_r_tma", "K3 k_sel_greedy"]
it = t[4:-2]  # drop the ends (graph launch boundaries show up as gaps anyway)
span = (it[:, :, 1] - it[:, :, 0]) / 1e3
print(f"config {cfg_id}: {len(it)} iterations, device-clock microseconds (median / mean)")
for j, nme in enumerate(names):
    nxt = it[:, j + 1, 0] if j < 3 else np.r_[it[1:, 0, 0], it[-1:, 0, 0]]
    gap = (nxt - it[:, j, 1]) / 1e3
    if j == 3:
        gap = gap[:-1]
    print(f"  {nme:16s} span {np.median(span[:, j]):8.2f} / {span[:, j].mean():8.2f}   "
          f"gap to next start {np.median(gap):7.2f} / {gap.mean():7.2f}")
period = (it[1:, 0, 0] - it[:-1, 0, 0]) / 1e3
print(f"  iteration period (K4 start to K4 start) {np.median(period):.2f} / {period.mean():.2f}")
