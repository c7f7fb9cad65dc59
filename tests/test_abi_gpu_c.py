"""The C ABI used from plain C on the GPU (tests/c/abi_gpu.c): lifecycle, a bitwise
fixed point, the wavespeed closed form and a deferred domain error."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_plain_c_gpu_consumer(tmp_path):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2104_08571_b200")
    exe = str(tmp_path / "abi_gpu")
    subprocess.check_call(["gcc", "-std=c11", "-O1", "-ffp-contract=off", "-Wall", "-Werror",
                           "-I", os.path.join(root, "include"),
                           os.path.join(root, "tests", "c", "abi_gpu.c"), "-L", libdir,
                           "-lripple_fv", f"-Wl,-rpath,{libdir}", "-lm", "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip() == "ok"
