"""bench.py contract on the GPU: one JSON line with the required keys, at N=1 and
(functional check) N=2 ranks sharing cuda:0 through torchrun + the P2P transport."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
        "gpu_launches", "clocks", "e2e"}


def _last_json(out):
    return json.loads(out.strip().splitlines()[-1])


def test_bench_single_gpu_line():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "5", "--warmup", "3",
                        "--no-cpu-baseline", "--e2e-steps", "2"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] == 5
    assert 0 < d["roofline"]["frac"] < 1.5


def test_bench_two_ranks_shared_device_p2p():
    env = dict(os.environ, RPL_SHARE_DEVICE="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        "29533", "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline", "--e2e-steps", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["config"]["parts"] == [1, 2]
    assert d["config"]["global_cells"] == [1024, 2048]
