"""Host-only tests of the C ABI (no GPU): exports, config validation, halo plan.

The halo plan is checked against the oracle: applying its edges to partitioned
copies of a random field must reproduce, cell for cell, the oracle's padded
global array ("halo soundness"), with every ghost written exactly
once.
"""
import ctypes
import itertools
import os
import re

import numpy as np
import pytest

import oracle
import paper_2104_08571_b200 as R
from paper_2104_08571_b200 import _native as N
import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "ripple_fv.h")).read()
    names = set(re.findall(r"\b(rpl_[a-z_0-9]+)\s*\(", hdr))
    assert len(names) >= 17
    lib = ctypes.CDLL(N.LIB_PATH)
    for n in sorted(names):
        assert hasattr(lib, n), n
    assert set(N.EXPORTS) == names


@pytest.mark.parametrize("kw,status", [
    (dict(size=(10, 8), parts=(3, 1)), -2),
    (dict(size=(10, 8), pad=0), -3),
    (dict(size=(10, 8), pad=5), -1),
    (dict(size=(10, 8), bc_lo=["periodic", "clamp"], bc_hi=["clamp", "clamp"]), -1),
    (dict(size=(10, 8), parts=(10, 1), pad=2), -1),     # partition extent < pad
    (dict(size=(10, 8), gamma=1.0), -1),
    (dict(size=(10, 8), nranks=3), -1),
    (dict(size=(16, 16), parts=(2, 2), nranks=4, rank=1), -1),  # missing nccl id
    (dict(size=(16, 16), parts=(2, 2), nranks=4, rank=1, nccl_id=b"x" * 128,
          transport="loopback"), -1),                           # loopback is one rank
])
def test_config_errors(kw, status):
    with pytest.raises(N.RplError) as ei:
        R.config_check(**kw)
    assert ei.value.status == status


def test_config_ok_and_arena():
    R.config_check(size=(1024, 1024), pad=2)
    R.config_check(size=(64, 64), parts=(2, 2), transport="loopback")
    R.config_check(size=(64, 64), parts=(2, 2), transport="loopback_nccl")
    n = R.arena_bytes(size=(1024, 1024), pad=2, dtype="f64")
    # two padded buffers, C=4 comps, pitch >= 1024 + ghosts, rows 1028
    assert 2 * 4 * 1028 * 1030 * 8 <= n <= 2 * 4 * 1028 * 1152 * 8 + 4096


def _bcs(kind, D):
    return [kind] * D


def _emulate(n, pad, parts, bc_lo, bc_hi, U):
    """Apply the library's halo plan in numpy; return per-partition padded arrays."""
    D = len(n)
    S = [n[d] // parts[d] for d in range(D)]
    plan = R.halo_plan(size=n, pad=pad, parts=parts, bc_lo=bc_lo, bc_hi=bc_hi)
    nparts = int(np.prod(parts))
    bufs, counts = {}, {}
    C = D + 2
    for p in range(nparts):
        pc = [p % parts[0], (p // parts[0]) % (parts[1] if D > 1 else 1),
              p // (parts[0] * (parts[1] if D > 1 else 1))][:D]
        lo = [pc[d] * S[d] for d in range(D)]
        B = np.full(tuple(S[d] + 2 * pad for d in reversed(range(D))) + (C,), np.nan)
        sl = tuple(slice(pad, pad + S[d]) for d in reversed(range(D)))
        gsl = tuple(slice(lo[d], lo[d] + S[d]) for d in reversed(range(D)))
        B[sl] = U[gsl]
        bufs[p] = (B, lo)
        counts[p] = np.zeros(B.shape[:-1], int)
    for e in plan:
        B, lo = bufs[e["dst_part"]]
        ranges = [range(e["dst_lo"][d], e["dst_hi"][d]) for d in range(D)]
        for t in itertools.product(*ranges):
            s = []
            for d in range(D):
                k = t[d] - e["dst_lo"][d]
                m = e["mode"][d]
                s.append(e["src_lo"][d] + k if m == N.MAP_TRANSLATE else
                         e["src_hi"][d] - 1 - k if m == N.MAP_REFLECT else e["src_lo"][d])
            v = U[tuple(reversed(s))].copy()
            for d in range(D):
                if e["mode"][d] == N.MAP_REFLECT:
                    v[1 + d] = -v[1 + d]
            idx = tuple(t[d] - lo[d] + pad for d in reversed(range(D)))
            B[idx] = v
            counts[e["dst_part"]][idx] += 1
    return bufs, counts, S


@pytest.mark.parametrize("n,parts,kind_lo,kind_hi", [
    ((12,), (3,), "clamp", "reflective"),
    ((12,), (4,), "periodic", "periodic"),
    ((8, 6), (1, 2), "clamp", "clamp"),
    ((8, 6), (2, 3), "periodic", "periodic"),
    ((8, 6), (2, 2), "reflective", "clamp"),
    ((6, 4, 4), (2, 2, 2), "clamp", "reflective"),
    ((6, 4, 4), (3, 1, 2), "periodic", "periodic"),
])
@pytest.mark.parametrize("pad", [1, 2])
def test_halo_plan_matches_oracle_ghost_fill(n, parts, kind_lo, kind_hi, pad):
    D = len(n)
    bl, bh = _bcs(kind_lo, D), _bcs(kind_hi, D)
    U = W.random_state(n, seed=11)
    bufs, counts, S = _emulate(n, pad, parts, bl, bh, U)
    kinds = {"clamp": oracle.BC_TRANSMISSIVE, "periodic": oracle.BC_PERIODIC,
             "reflective": oracle.BC_REFLECTIVE}
    g = oracle.Grid(n, pad=pad, bc_lo=[kinds[k] for k in bl], bc_hi=[kinds[k] for k in bh])
    P = np.zeros(oracle.padded_shape(g))
    P[tuple(slice(pad, pad + n[d]) for d in reversed(range(D)))] = U
    P = oracle.fill_ghosts(g, P)
    for p, (B, lo) in bufs.items():
        gsl = tuple(slice(lo[d], lo[d] + S[d] + 2 * pad) for d in reversed(range(D)))
        assert np.array_equal(B, P[gsl]), p  # NaN-free and equal
        interior = np.zeros(counts[p].shape, bool)
        interior[tuple(slice(pad, pad + S[d]) for d in reversed(range(D)))] = True
        assert np.all(counts[p][~interior] == 1)
        assert np.all(counts[p][interior] == 0)


def test_halo_plan_edge_counts_slabs():
    # 1-D, 4 partitions, clamp: 6 exchange edges between partitions
    plan = R.halo_plan(size=(16,), pad=2, parts=(4,))
    xch = [e for e in plan if e["src_part"] != e["dst_part"]]
    assert len(xch) == 6
    plan1 = R.halo_plan(size=(16,), pad=2, parts=(1,))
    assert all(e["src_part"] == e["dst_part"] for e in plan1)


def test_order2_config_checks():
    """order 2 needs pad >= 2 (stencil radius 2); order must be 1 or 2 (host only)."""
    from paper_2104_08571_b200 import _native as N
    R.config_check(size=(64, 32), pad=2, order=2)
    with pytest.raises(N.RplError) as e:
        R.config_check(size=(64, 32), pad=1, order=2)
    assert "RPL_E_PAD_TOO_SMALL" in str(e.value)
    with pytest.raises(N.RplError):
        R.config_check(size=(64, 32), pad=2, order=3)


def test_plain_c_consumer(tmp_path):
    """The boundary is a C ABI: a plain C program (tests/c/abi_host.c) compiled with gcc
    against include/ripple_fv.h and linked to libripple_fv.so uses the host-only calls."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2104_08571_b200")
    exe = str(tmp_path / "abi_host")
    subprocess.check_call(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
                           os.path.join(root, "tests", "c", "abi_host.c"), "-L", libdir,
                           "-lripple_fv", f"-Wl,-rpath,{libdir}", "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip() == "ok"


def test_kernel_name_binding_returns_string():
    """rpl_kernel_name returns a C string (bytes through ctypes), "" for a null domain."""
    from paper_2104_08571_b200 import _native as N
    assert N.lib().rpl_kernel_name(None, 0) == b""
    assert N.lib().rpl_kernel_name(None, 1) == b""
