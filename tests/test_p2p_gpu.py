"""Multi-rank path on one GPU: 2-4 processes (one partition each) share cuda:0 and
exchange halos through the P2P transport (CUDA IPC peer mappings written directly
by the step kernels + system-scope flag kernel), with a gloo process group only
for the IPC-handle all-gather.  Result must be bitwise equal to the single-rank
run (BASELINE.json north_star: bit-identical across GPU counts)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, n, parts, kw, steps, q, t_end=None, env=None):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(env or {})
    import torch
    import torch.distributed as dist

    import paper_2104_08571_b200 as R
    import workloads as W
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        D = len(n)
        dx = [1.0 / n[0]] * D
        dom = R.Domain(n, parts=parts, nranks=world, rank=rank, transport="p2p", dx=dx, **kw)
        blob = dom.p2p_export()
        blobs = [None] * world
        dist.all_gather_object(blobs, blob)
        dom.p2p_attach(blobs)
        U = W.shock_bubble(n, dx=dx, box=(dom.lo, dom.hi))
        if kw.get("dtype") == "f32":
            U = U.astype(np.float32)
        dom.set_state(U)
        if t_end is None:
            s = dom.max_wavespeed()
            dom.advance(0.4 * dx[0] / s, steps)
        else:
            s = dom.advance_to(t_end)   # (t reached, steps taken)
        out = dom.get_state()
        q.put((rank, dom.lo, dom.hi, out, s))
        dom.close()
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _single(n, kw, steps, t_end=None):
    import paper_2104_08571_b200 as R
    import workloads as W
    D = len(n)
    dx = [1.0 / n[0]] * D
    U = W.shock_bubble(n, dx=dx)
    if kw.get("dtype") == "f32":
        U = U.astype(np.float32)
    with R.Domain(n, dx=dx, **kw) as dom:
        dom.set_state(U)
        if t_end is None:
            s = dom.max_wavespeed()
            dom.advance(0.4 * dx[0] / s, steps)
        else:
            s = dom.advance_to(t_end)
        return dom.get_state(), s


@pytest.mark.parametrize("n,parts,kw", [
    ((130, 64), (1, 2), {}),
    ((128, 96), (2, 1), dict(bc_lo=["periodic", "reflective"], bc_hi=["periodic", "clamp"])),
    ((40, 32, 24), (1, 1, 2), dict(dtype="f32")),
    ((40, 32, 24), (2, 2, 1), {}),
])
def test_p2p_ranks_bitwise_equal_single_rank(n, parts, kw):
    _check(n, parts, kw, None)


@pytest.mark.parametrize("n,parts,kw", [
    ((130, 64), (1, 2), {}),
    ((130, 64), (2, 2), dict(kernel="split")),
    ((40, 32, 24), (1, 1, 2), {}),
])
def test_p2p_device_cfl_bitwise_equal_single_rank(n, parts, kw):
    """rpl_advance_to over ranks: the wavespeed slot rides the P2P step sync."""
    _check(n, parts, kw, 0.02)


@pytest.mark.parametrize("n,parts,kw", [
    ((130, 64), (1, 2), dict(order=2)),
    ((40, 32, 24), (1, 2, 2), dict(order=2)),
    ((40, 32, 24), (1, 1, 2), dict(order=2, kernel="split")),
])
def test_p2p_order2_bitwise_equal_single_rank(n, parts, kw):
    """Order 2 (radius-2 halos; in 3-D two passes per step) over P2P ranks."""
    _check(n, parts, kw, None)


@pytest.mark.parametrize("n,parts,kw", [
    ((128, 96), (1, 8), {}),
    ((40, 32, 24), (2, 2, 2), dict(dtype="f32")),
])
def test_p2p_eight_ranks_bitwise_equal_single_rank(n, parts, kw):
    """8 ranks (the north star's largest GPU count), y-slabs and a 2x2x2 block grid."""
    _check(n, parts, kw, None)




def _stall_rank(rank, port, q):
    """Rank 1 attaches and then never steps; rank 0 steps and must get an error from
    the bounded P2P wait (RPL_P2P_TIMEOUT_S) instead of hanging."""
    import sys
    import time
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["RPL_P2P_TIMEOUT_S"] = "2"
    import torch
    import torch.distributed as dist

    import paper_2104_08571_b200 as R
    import workloads as W
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        torch.cuda.set_device(0)
        n = (64, 64)
        dom = R.Domain(n, parts=(1, 2), nranks=2, rank=rank, transport="p2p")
        blobs = [None] * 2
        dist.all_gather_object(blobs, dom.p2p_export())
        dom.p2p_attach(blobs)
        if rank == 0:
            dom.set_state(W.random_state(n, box=(dom.lo, dom.hi)))  # no peer sync here
            t0 = time.time()
            err = None
            try:
                dom.advance(1e-4, 1)
                dom.synchronize()
            except R.RplError as e:
                err = str(e)
            q.put((err, time.time() - t0))
        dist.barrier()  # rank 1 idles here until rank 0 is done
        dom.close()
    finally:
        dist.destroy_process_group()


def test_p2p_stalled_peer_times_out():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_stall_rank, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err, dt = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert err is not None and "P2P" in err, err
    assert dt < 60


def _run_ranks(n, parts, kw, t_end, steps=6, env=None):
    world = int(np.prod(parts))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, n, parts, kw, steps, q, t_end, env))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    return res


def _check(n, parts, kw, t_end):
    steps = 6
    res = _run_ranks(n, parts, kw, t_end, steps)
    ref, s_ref = _single(n, kw, steps, t_end)
    D = len(n)
    for rank, lo, hi, out, s in res:
        assert s == s_ref
        sl = tuple(slice(lo[d], hi[d]) for d in reversed(range(D)))
        assert np.array_equal(out, ref[sl]), rank


@pytest.mark.parametrize("n,parts,kw", [((130, 64), (1, 2), {}), ((40, 32, 24), (2, 2, 1), {})])
def test_p2p_fault_hook_turns_bitwise_test_red(n, parts, kw):
    """RPL_FAULT_HALO=1 flips one mantissa bit of one halo ghost per rank after every
    exchange: the rank-vs-single bit-identity check must then fail (it is not blind)."""
    steps = 6
    res = _run_ranks(n, parts, kw, None, steps, env={"RPL_FAULT_HALO": "1"})
    ref, _ = _single(n, kw, steps)
    D = len(n)
    same = [np.array_equal(out, ref[tuple(slice(lo[d], hi[d]) for d in reversed(range(D)))])
            for _, lo, hi, out, _ in res]
    assert not all(same)
