"""bench.py's N > 1 path (points sharded over ranks) end to end
on one GPU: two torchrun ranks pinned to cuda:0 with the gloo backend
(CRISP_BENCH_DEVICE; no GPU kernel waits on another rank).  Guaranteed Mode
with the exact global fallback and Optimized Mode with global patience must
give the single-index recall for every G;
the JSON line must follow the driver contract."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--steps", "2", "--warmup", "3", "--N", "120000", "--Q", "1500", "--no-cpu-baseline"]


def _line(out):
    return json.loads(out.strip().splitlines()[-1])


def test_bench_two_ranks_match_one():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    one = subprocess.run([sys.executable, "bench.py", *ARGS], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert one.returncode == 0, one.stderr[-2000:]
    env = dict(os.environ, CRISP_BENCH_DEVICE="0")
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29561", "bench.py", "--gpus", "2", *ARGS],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert two.returncode == 0, two.stderr[-2000:]
    a, b = _line(one.stdout), _line(two.stdout)
    assert a["n_gpus"] == 1 and b["n_gpus"] == 2
    for key in ("metric", "value", "unit", "ms_per_step", "higher_is_better", "scaling", "roofline", "clocks", "e2e"):
        assert key in b
    assert b["e2e"]["value"] > 0 and b["e2e"]["h2d_bytes_per_step"] > 0  # end to end at N = 2 too
    # phi=0 with the exact global fallback, phi=1 with the patience rule over the global
    # (h, gid) order: both identical to the single index
    assert b["per_mode"]["guaranteed"]["recall"] == a["per_mode"]["guaranteed"]["recall"]
    assert b["per_mode"]["optimized"]["recall"] == a["per_mode"]["optimized"]["recall"]
