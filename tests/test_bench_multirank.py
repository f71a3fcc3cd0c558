"""bench.py's N > 1 control flow on CPU: `bench.py --gpus 2` re-launches itself under
torch.distributed.run (gloo here), shards frames (weak: a batch per rank; strong: one batch
split by shard.frame_range), takes the max over ranks and prints one line from rank 0 with
n_gpus = 2.  --stub replaces the kernel with a torch op and CUDA events with wall clock
(a control-flow check, never a measurement)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _run(*extra):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="", OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--stub", "--steps", "2", "--warmup",
                        "1", "--no-cpu", "--no-sweep", "--no-parity", *extra],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    assert "spawning 2 ranks" in r.stderr and "world 2" in r.stderr
    return json.loads(lines[0])


@pytest.mark.parametrize("scaling,frames,shards", [("weak", 128, [[0, 64], [0, 64]]),
                                                    ("strong", 64, [[0, 32], [32, 64]])])
def test_bench_two_ranks(scaling, frames, shards):
    d = _run("--scaling", scaling)
    assert d["n_gpus"] == 2 and d["scaling"] == scaling
    assert d["config"]["frames_per_step"] == frames
    assert d["config"]["frame_shards"] == shards
    assert d["config"]["pixel_fits_per_step"] == frames * 64 * 48 * 2
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert "STUB" in d["data"]
