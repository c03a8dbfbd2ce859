"""bench.py's command-line contract on a box without GPUs (no compute).

* `--gpus N` must never be measured on fewer GPUs: outside torchrun the script
  re-launches itself as N ranks and refuses when fewer devices are visible; under
  torchrun WORLD_SIZE must equal --gpus ("bench.py --gpus N is
  ignored by the GPU arm").
* the byte counts the roofline is computed from are SURVEY §8(d)'s formulas.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                          text=True, env=e, timeout=300)


def _no_gpu():
    import torch

    return torch.cuda.device_count() == 0


@pytest.mark.skipif(not _no_gpu(), reason="needs a box without GPUs")
def test_gpus_n_refuses_to_measure_fewer_devices():
    out = _run(["--gpus", "2", "--steps", "3", "--warmup", "3"])
    assert out.returncode == 2
    assert "refusing to measure fewer GPUs" in out.stderr
    assert '"n_gpus"' not in out.stdout  # no line at all, in particular no n_gpus: 1


def test_world_size_must_match_gpus():
    out = _run(["--gpus", "4", "--steps", "3", "--warmup", "3"],
               env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert out.returncode == 2
    assert "WORLD_SIZE=2 but --gpus 4" in out.stderr
    assert out.stdout.strip() == ""


def test_algorithmic_bytes_are_the_survey_formulas():
    import bench

    c3, c5 = bench.CONFIGS[3], bench.CONFIGS[5]
    # K2: 16·m·n + 8·(2m + n)  (SURVEY §8(d) "Roofline definition")
    assert bench.k2_bytes(c3) == 16 * 8192 * 8192 + 8 * (2 * 8192 + 8192) == 1073938432
    assert bench.k2_bytes(c5) == 34361049088
    assert bench.k2_bytes(c5, world=8) == 16 * 8192 * 32768 + 8 * (2 * 8192 + 32768)
    # iteration: + 16·q·n (two passes over B) + 16·p·q (X) + 8·p·q (X_ref) + 8·m (cached G row)
    it3 = bench.iteration_bytes(c3, gram_cached=True, track_ref=True)
    assert it3 == 1073938432 + 16 * 2048 * 8192 + 24 * 2048 * 2048 + 8 * 8192 == 1443102720
