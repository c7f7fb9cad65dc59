"""The C ABI used from plain C on the GPU (tests/c/abi_gpu.c): lifecycle, a bitwise
fixed point, the wavespeed closed form, a deferred domain error, and a 30-step run
of a random state over 3 partitions vs the oracle's C API (<= 1e-10, S15) and vs
the split kernel (bitwise)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_plain_c_gpu_consumer(tmp_path):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2104_08571_b200")
    import oracle
    orcdir = os.path.dirname(oracle.build())
    exe = str(tmp_path / "abi_gpu")
    subprocess.check_call(["gcc", "-std=c11", "-O1", "-ffp-contract=off", "-Wall", "-Werror",
                           "-I", os.path.join(root, "include"), "-I", orcdir,
                           os.path.join(root, "tests", "c", "abi_gpu.c"), "-L", libdir,
                           "-lripple_fv", f"-Wl,-rpath,{libdir}",
                           os.path.join(orcdir, "liboracle.so"), f"-Wl,-rpath,{orcdir}",
                           "-lm", "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip() == "ok"
