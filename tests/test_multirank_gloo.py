"""N > 1 path on CPU: two processes (gloo, world_size 2) run the library's halo
plan exactly as the NCCL exchange does -- pack every edge whose source partition
is mine and destination is the peer's into one message per peer (plan order),
send/recv, unpack -- and check that every ghost of every rank's partition equals
the oracle's single-block ghost fill.  This checks the message
layout the NCCL transport's peer lists use (the plan's edges in plan order, one
message per peer) on CPU, with the host re-implementing pack and unpack.  The
library's own device path -- shell tiles, the side stream, the batched pack
(`k_edges`) and unpack kernels, the events -- runs on one GPU through the LOOPBACK
transport (tests/test_loopback_gpu.py, bitwise vs one partition); only the
ncclSend/ncclRecv calls themselves need two GPUs.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2104_08571_b200 as R
from paper_2104_08571_b200 import _native as N
import workloads as W

KIND = {"clamp": oracle.BC_TRANSMISSIVE, "periodic": oracle.BC_PERIODIC,
        "reflective": oracle.BC_REFLECTIVE}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _src_index(e, t, D):
    s = []
    for d in range(D):
        k = t[d] - e["dst_lo"][d]
        m = e["mode"][d]
        s.append(e["src_lo"][d] + k if m == N.MAP_TRANSLATE else
                 e["src_hi"][d] - 1 - k if m == N.MAP_REFLECT else e["src_lo"][d])
    return s


def _box_cells(e, D):
    ext = [e["dst_hi"][d] - e["dst_lo"][d] for d in range(D)]
    for i in range(int(np.prod(ext))):
        t, r = [], i
        for d in range(D):  # x fastest, like k_edge
            t.append(e["dst_lo"][d] + r % ext[d])
            r //= ext[d]
        yield t


def _worker(rank, world, port, n, parts, bl, bh, pad, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        D = len(n)
        S = [n[d] // parts[d] for d in range(D)]
        C = D + 2
        U = W.random_state(n, seed=31)  # global field (test only)
        plan = R.halo_plan(size=n, pad=pad, parts=parts, bc_lo=bl, bc_hi=bh)
        pc = [rank % parts[0], (rank // parts[0]) % (parts[1] if D > 1 else 1),
              rank // (parts[0] * (parts[1] if D > 1 else 1))][:D]
        lo = [pc[d] * S[d] for d in range(D)]
        B = np.full(tuple(S[d] + 2 * pad for d in reversed(range(D))) + (C,), np.nan)
        B[tuple(slice(pad, pad + S[d]) for d in reversed(range(D)))] = \
            U[tuple(slice(lo[d], lo[d] + S[d]) for d in reversed(range(D)))]

        def local(e):  # my interior -> value at source index (only my cells are readable)
            return True

        send, recv = {}, {}
        for e in plan:
            if e["src_part"] == rank and e["dst_part"] != rank:
                send.setdefault(e["dst_part"], []).append(e)
            if e["dst_part"] == rank and e["src_part"] != rank:
                recv.setdefault(e["src_part"], []).append(e)

        def read_mine(s):
            li = tuple(s[d] - lo[d] + pad for d in reversed(range(D)))
            assert all(0 <= s[d] - lo[d] < S[d] for d in range(D)), "source not in my interior"
            return B[li]

        # pack: per peer, edges in plan order, each edge [C][count] (k_edge layout)
        reqs = []
        bufs = {}
        for peer, edges in sorted(send.items()):
            chunks = []
            for e in edges:
                vals = []
                for t in _box_cells(e, D):
                    v = read_mine(_src_index(e, t, D)).copy()
                    for d in range(D):
                        if e["mode"][d] == N.MAP_REFLECT:
                            v[1 + d] = -v[1 + d]
                    vals.append(v)
                chunks.append(np.array(vals).T.ravel())
            bufs[peer] = torch.from_numpy(np.concatenate(chunks))
            reqs.append(dist.isend(bufs[peer], peer))
        got = {}
        for peer, edges in sorted(recv.items()):
            cnt = sum(int(np.prod([e["dst_hi"][d] - e["dst_lo"][d] for d in range(D)])) * C
                      for e in edges)
            got[peer] = torch.empty(cnt, dtype=torch.float64)
            reqs.append(dist.irecv(got[peer], peer))
        for r in reqs:
            r.wait()
        # local edges (physical BCs of my partition)
        for e in plan:
            if e["src_part"] == rank and e["dst_part"] == rank:
                for t in _box_cells(e, D):
                    v = read_mine(_src_index(e, t, D)).copy()
                    for d in range(D):
                        if e["mode"][d] == N.MAP_REFLECT:
                            v[1 + d] = -v[1 + d]
                    B[tuple(t[d] - lo[d] + pad for d in reversed(range(D)))] = v
        # unpack
        for peer, edges in sorted(recv.items()):
            msg = got[peer].numpy()
            off = 0
            for e in edges:
                cells = list(_box_cells(e, D))
                arr = msg[off: off + C * len(cells)].reshape(C, len(cells))
                off += C * len(cells)
                for i, t in enumerate(cells):
                    B[tuple(t[d] - lo[d] + pad for d in reversed(range(D)))] = arr[:, i]
        g = oracle.Grid(n, pad=pad, bc_lo=[KIND[k] for k in bl], bc_hi=[KIND[k] for k in bh])
        P = np.zeros(oracle.padded_shape(g))
        P[tuple(slice(pad, pad + n[d]) for d in reversed(range(D)))] = U
        P = oracle.fill_ghosts(g, P)
        ref = P[tuple(slice(lo[d], lo[d] + S[d] + 2 * pad) for d in reversed(range(D)))]
        q.put((rank, bool(np.array_equal(B, ref)), int(np.isnan(B).sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,parts,bl,bh", [
    ((10, 8), (1, 2), ["clamp", "reflective"], ["reflective", "clamp"]),
    ((10, 8), (2, 1), ["periodic", "clamp"], ["periodic", "clamp"]),
    ((6, 4, 8), (1, 1, 2), ["reflective", "periodic", "periodic"],
     ["clamp", "periodic", "periodic"]),
])
def test_two_rank_halo_exchange_gloo(n, parts, bl, bh):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, parts, bl, bh, 2, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, nans in res:
        assert nans == 0, (rank, nans)
        assert ok, rank
