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
    """The default run: BASELINE configs[2] (512^3 fp64) as the headline, configs[3]
    and configs[1] as extra keys, each with its own roofline and step kernel."""
    r = subprocess.run([sys.executable, "bench.py", "--steps", "5", "--warmup", "3",
                        "--extra-steps", "5", "--no-cpu-baseline", "--e2e-steps", "2"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] == 5
    assert 0 < d["roofline"]["frac"] < 1.5
    assert d["config"]["global_cells"] == [512, 512, 512] and d["dtype"] == "f64"
    assert d["roofline"]["kernel"].startswith("k_step3d")
    assert d["halo"]["exposed_ms_per_step"] is None  # N = 1: no exchange
    assert set(d["extra"]) == {"w384", "2d1024"}
    for k, x in d["extra"].items():
        assert x["value"] > 0 and 0 < x["roofline"]["frac"] < 1.5, k
    assert d["extra"]["w384"]["dtype"] == "f32"
    assert d["extra"]["2d1024"]["roofline"]["kernel"].startswith("k_step2d_ra")


def test_bench_two_ranks_shared_device_p2p():
    env = dict(os.environ, RPL_SHARE_DEVICE="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        "29533", "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--workload", "2d1024", "--no-cpu-baseline", "--e2e-steps", "1"],
                       cwd=ROOT, capture_output=True,
                       text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["config"]["parts"] == [1, 2]
    assert d["config"]["global_cells"] == [2048, 1024]
    h = d["halo"]
    assert h["event_ms_per_step"] is not None and h["differential_ms_per_step"] is not None
    assert h["exchanges_per_step"] == 1


def test_bench_gpus_flag_relaunches_ranks():
    """`python bench.py --gpus 2` (no torchrun environment) launches 2 ranks itself and
    rank 0 reports n_gpus = 2 (here both ranks share cuda:0: a functional check)."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["RPL_SHARE_DEVICE"] = "1"
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup",
                        "3", "--workload", "w384", "--no-cpu-baseline", "--e2e-steps", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["config"]["parts"] == [2, 1, 1]
    assert d["config"]["global_cells"] == [768, 384, 384]
