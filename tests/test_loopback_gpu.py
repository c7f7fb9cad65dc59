"""The NCCL transport's choreography on one GPU (RPL_TRANSPORT_LOOPBACK, include/
ripple_fv.h): the local partitions exchange halos only through the message path --
shell tiles of the fused step kernel first, then on a high-priority side stream one
pack kernel over every edge, the transfer (a device copy where NCCL would send/recv)
and one unpack kernel, overlapped with the interior tiles; the next step waits on
the halo event only (north_star: "only boundary cells wait on communication").
Bitwise equal to one partition (north_star: the exchange must not change the
arithmetic).  The NCCL calls themselves need a second GPU."""
import numpy as np
import pytest

import paper_2104_08571_b200 as R
import workloads as W
from test_parity_gpu import bits_equal, run_gpu

pytestmark = pytest.mark.gpu


def _lb(U0, dt, steps, **kw):
    return run_gpu(U0, dt, steps, transport="loopback", **kw)


@pytest.mark.parametrize("n,parts", [((190, 126), (1, 3)), ((190, 126), (2, 3)),
                                     ((130, 64), (2, 1))])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_loopback_2d_bitwise(n, parts, dtype):
    dx = [1.0 / n[0]] * 2
    U0 = W.shock_bubble(n, dx=dx)
    if dtype == "f32":
        U0 = U0.astype(np.float32)
    dt = 0.4 * dx[0] / 5.8
    ref = run_gpu(U0, dt, 7, dtype=dtype, dx=dx)
    assert bits_equal(_lb(U0, dt, 7, dtype=dtype, dx=dx, parts=parts), ref)


@pytest.mark.parametrize("n,parts,kw", [
    ((40, 33, 48), (1, 1, 2), {}),
    ((40, 33, 48), (1, 1, 4), dict(dtype="f32")),
    ((64, 32, 24), (2, 2, 2), {}),
    ((64, 32, 24), (2, 2, 2), dict(dtype="f32", bc_lo=["periodic", "reflective", "clamp"],
                                   bc_hi=["periodic", "clamp", "reflective"])),
    ((64, 32, 24), (2, 1, 1), dict(layout="aos")),
])
def test_loopback_3d_bitwise(n, parts, kw):
    dx = [1.0 / n[0]] * 3
    U0 = W.shock_bubble(n, dx=dx)
    dtype = kw.get("dtype", "f64")
    if dtype == "f32":
        U0 = U0.astype(np.float32)
    dt = 0.4 * dx[0] / 5.8
    kw = dict(kw)
    kw.pop("dtype", None)
    bcs = {k: kw[k] for k in ("bc_lo", "bc_hi") if k in kw}
    ref = run_gpu(U0, dt, 6, dtype=dtype, dx=dx, rows_per_chunk=8, **bcs)
    got = _lb(U0, dt, 6, dtype=dtype, dx=dx, parts=parts, rows_per_chunk=8, **kw)
    assert bits_equal(got, ref)


@pytest.mark.parametrize("kw", [dict(kernel="split"), dict(order=2), dict(order=2, kernel="split")])
def test_loopback_non_overlapped_paths_bitwise(kw):
    """Split kernels and order 2 exchange after the whole step (no tile lists)."""
    n = (64, 40, 24)
    dx = [1.0 / n[0]] * 3
    U0 = W.shock_bubble(n, dx=dx)
    dt = 0.4 * dx[0] / 5.8
    ref = run_gpu(U0, dt, 4, dx=dx, **kw)
    assert bits_equal(_lb(U0, dt, 4, dx=dx, parts=(1, 2, 2), **kw), ref)


def test_loopback_device_cfl_bitwise():
    n = (130, 64)
    dx = [1.0 / n[0]] * 2
    U0 = W.shock_bubble(n, dx=dx)
    out = []
    for kw in ({}, dict(parts=(2, 2), transport="loopback")):
        with R.Domain(n, dx=dx, **kw) as dom:
            dom.set_state(U0)
            t, k = dom.advance_to(0.01)
            out.append((dom.get_state(), t, k))
    assert out[0][1:] == out[1][1:] and bits_equal(out[0][0], out[1][0])


def test_loopback_launches_and_halo_events():
    """Per step: shell + interior launch per partition, one pack and one unpack kernel;
    rpl_profile_halo sees one exchange per step."""
    n = (64, 32, 48)
    dx = [1.0 / n[0]] * 3
    U0 = W.shock_bubble(n, dx=dx)
    with R.Domain(n, dx=dx, parts=(1, 1, 2), transport="loopback", rows_per_chunk=8) as dom:
        dom.set_state(U0)
        assert dom.launches_per_step == 2 * 2 + 2
        dom.profile(64)
        dom.advance(1e-4, 3)
        ms, n_k = dom.profile_read()
        hms, nx = dom.profile_halo()
        assert n_k == 3 * 4 and nx == 3 and hms >= 0.0
        assert dom.kernel_name() == "k_step3d_sp<pd>"


def test_loopback_fault_hook_turns_red(monkeypatch):
    n = (190, 126)
    dx = [1.0 / n[0]] * 2
    U0 = W.shock_bubble(n, dx=dx)
    dt = 0.4 * dx[0] / 5.8
    ref = run_gpu(U0, dt, 5, dx=dx)
    monkeypatch.setenv("RPL_FAULT_HALO", "1")
    assert not np.array_equal(_lb(U0, dt, 5, dx=dx, parts=(2, 3)), ref)


@pytest.mark.parametrize("n,parts,kw", [
    ((200,), (4,), dict(bc_lo=["periodic"], bc_hi=["periodic"])),   # 1-D: split kernel
    ((130, 64), (2, 2), dict(pad=1)),                               # pad 1 (one ghost layer)
    ((130, 64), (1, 4), dict(order=2)),                             # order 2 in 2-D
    ((40, 33, 48), (1, 1, 8), dict(dtype="f32")),                   # 8 thin z-slabs
])
def test_loopback_more_shapes_bitwise(n, parts, kw):
    D = len(n)
    dx = [1.0 / n[0]] * D
    U0 = W.random_state(n, seed=47)
    kw = dict(kw)
    dtype = kw.pop("dtype", "f64")
    if dtype == "f32":
        U0 = U0.astype(np.float32)
    dt = 0.2 * dx[0] / 3.0
    ref = run_gpu(U0, dt, 5, dtype=dtype, dx=dx, **kw)
    assert bits_equal(_lb(U0, dt, 5, dtype=dtype, dx=dx, parts=parts, **kw), ref)


@pytest.mark.parametrize("n,parts,kw", [
    ((190, 126), (2, 3), {}),                       # 2-D, overlapped (shell / side stream)
    ((64, 32, 24), (2, 2, 2), dict(dtype="f32")),   # 3-D blocks, overlapped
    ((64, 40, 24), (1, 2, 2), dict(order=2)),       # order 2: exchange after the step
])
def test_loopback_nccl_send_recv_bitwise(n, parts, kw):
    """RPL_TRANSPORT_LOOPBACK_NCCL: the halo messages travel through grouped
    ncclSend/ncclRecv to self on a one-rank communicator (maxCTAs config) -- the NCCL
    calls of the multi-rank transport, on one GPU -- bitwise equal to one partition."""
    D = len(n)
    dx = [1.0 / n[0]] * D
    U0 = W.shock_bubble(n, dx=dx)
    kw = dict(kw)
    dtype = kw.pop("dtype", "f64")
    if dtype == "f32":
        U0 = U0.astype(np.float32)
    dt = 0.4 * dx[0] / 5.8
    ref = run_gpu(U0, dt, 5, dtype=dtype, dx=dx, **kw)
    got = run_gpu(U0, dt, 5, dtype=dtype, dx=dx, parts=parts, transport="loopback_nccl", **kw)
    assert bits_equal(got, ref)
