"""bench.py's reference arm (--impl reference = the CPU oracle) runs without a
GPU: one JSON line with the contract's keys, under torchrun only rank 0 prints."""
import json
import os
import subprocess
import sys

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
