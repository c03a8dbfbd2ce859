"""Config 5's literal budget (10⁴ iterations, refresh every 1000) split into its parts:
device time of every 1000-iteration segment and of every refresh checkpoint, with the
SM clock sampled alongside (sustained power-capped operation, not the burst clocks of a
200-step window).  Prints one line per segment and a JSON summary."""
import json
import subprocess
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2408_05444_b200 as axb
from bench import CONFIGS, make_inputs_device, solver_config

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 5]
segs = int(sys.argv[2]) if len(sys.argv) > 2 else 10
A, B, Cm, X0, Xs = make_inputs_device(cfg, 1000, 0)
s = axb.Solver(A, B, Cm, X0, solver_config(axb, Xs, 10 ** 9), axb.Options(spectral_max_iter=200000))
del A, B, Cm
torch.cuda.empty_cache()
s.steps(10)


def clock():
    out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip().split(",")
    return float(out[0]), float(out[1])


it_ms, ck_ms = [], []
for seg in range(segs):
    s.steps(1000, mirror_refresh=False)
    it = s.last_timing()["loop_ms"]
    c_it = clock()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.checkpoint()
    torch.cuda.synchronize()
    ck = (time.perf_counter() - t0) * 1e3
    c_ck = clock()
    it_ms.append(it)
    ck_ms.append(ck)
    print(f"segment {seg}: 1000 iterations {it:.1f} ms ({1e6 / it:.1f} it/s), checkpoint {ck:.1f} ms; "
          f"SM {c_it[0]:.0f} MHz {c_it[1]:.0f} W after the iterations, {c_ck[0]:.0f} MHz after the checkpoint",
          flush=True)
tot = sum(it_ms) + sum(ck_ms)
print(json.dumps({"config": cfg["desc"], "segments": segs, "iterations_ms": [round(x, 1) for x in it_ms],
                  "checkpoint_ms": [round(x, 1) for x in ck_ms], "total_s": round(tot / 1e3, 2),
                  "it_per_s_with_refresh": round(1000 * segs / (tot / 1e3), 2),
                  "checkpoint_share": round(sum(ck_ms) / tot, 4)}))
