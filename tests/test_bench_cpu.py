"""bench.py's reference arm (--impl reference = the CPU oracle) runs without a
GPU: one JSON line with the contract's keys, under torchrun only rank 0 prints."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    r = subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, capture_output=True,
                       text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout


def test_reference_arm_json_line():
    out = _run(["--impl", "reference", "--workload", "2d1024", "--steps", "1", "--warmup", "0"])
    lines = [l for l in out.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["metric"] == "Gcell-updates/s" and d["higher_is_better"] is True


def test_reference_arm_other_ranks_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], env=env)
    assert not [l for l in out.strip().splitlines() if l.startswith("{")]


def test_gpus_flag_relaunches_under_torchrun():
    """--gpus 2 without a torchrun environment re-launches bench.py under
    torch.distributed.run with 2 ranks; rank 0 alone prints one line (reference arm: no
    GPU needed, so the launch path itself is exercised here)."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = _run(["--impl", "reference", "--workload", "2d1024", "--gpus", "2", "--steps", "1",
                "--warmup", "0"], env=env)
    lines = [l for l in out.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"


@pytest.mark.parametrize("wl", ["fd1k", "cfl1024", "o2_1024"])
def test_reference_arm_runs_the_workload_op(wl):
    """The reference arm times the same operation as the GPU arm (flux difference, CFL
    run, order-2 step), not always the order-1 step."""
    out = _run(["--impl", "reference", "--workload", wl, "--steps", "1", "--warmup", "0"])
    d = json.loads([l for l in out.strip().splitlines() if l.startswith("{")][0])
    op = {"fd1k": "fluxdiff", "cfl1024": "cfl", "o2_1024": "step"}[wl]
    assert f"op={op}" in d["config"]["sample"] and d["value"] > 0
    if wl == "fd1k":
        assert d["unit"] == "Gcell/s"


def test_weak_2d_decomposition_grows_x_and_y():
    """2-D weak scaling as the paper runs it: per-GPU size fixed, the
    domain grows in x and y, split along y."""
    import bench
    for n in (1, 2, 4, 8):
        gn, parts = bench.decomposition(bench.WORKLOADS["2d1024"], n)
        assert parts == [1, n] and gn[0] * gn[1] == n * 1024 * 1024 and gn[1] % n == 0
    assert bench.decomposition(bench.WORKLOADS["2d1024"], 4)[0] == [2048, 2048]
