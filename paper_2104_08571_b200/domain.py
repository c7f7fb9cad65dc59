"""Python binding of the rpl_* C ABI: same operations, argument marshalling only.

    create an N-D tensor with sizes, padding width and partition count  -> Domain(...)
    set the initial state                                                -> Domain.set_state
    fill the padding                                                     -> Domain.fill_padding
    advance by dt over n steps                                           -> Domain.advance
    read back the state                                                  -> Domain.get_state
(BASELINE.json north_star; include/ripple_fv.h.)  Every step runs in the CUDA
kernels of libripple_fv.so; this module never computes any part of the scheme.

Host arrays: numpy, either the dense AoS interior (nz, ny, nx, C) used by the
workloads/oracle side (converted here to the ABI's dense SoA (C, nz, ny, nx)),
or raw host pointers for zero-copy callers (``*_ptr`` methods).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N

_BC = {"transmissive": N.BC_TRANSMISSIVE, "clamp": N.BC_TRANSMISSIVE,
       "periodic": N.BC_PERIODIC, "reflective": N.BC_REFLECTIVE}


def _bc(v):
    return _BC[v] if isinstance(v, str) else int(v)


def make_config(size, pad=2, parts=None, dtype="f64", layout="soa", kernel="fused", gamma=1.4,
                dx=None, bc_lo=None, bc_hi=None, nranks=1, rank=0, nccl_id=None, device=0,
                stream=None, arena=None, rows_per_chunk=0, transport="nccl", order=1):
    size = [int(v) for v in size]
    D = len(size)
    if not 1 <= D <= 3:
        raise ValueError("ndim must be 1..3")
    cfg = N.Config()
    N.lib().rpl_config_init(ctypes.byref(cfg))
    cfg.ndim = D
    for d in range(3):
        cfg.size[d] = size[d] if d < D else 1
        cfg.parts[d] = (parts[d] if parts is not None else 1) if d < D else 1
        cfg.dx[d] = (dx[d] if dx is not None else 1.0 / size[d]) if d < D else 1.0
        cfg.bc_lo[d] = _bc(bc_lo[d]) if (bc_lo is not None and d < D) else N.BC_TRANSMISSIVE
        cfg.bc_hi[d] = _bc(bc_hi[d]) if (bc_hi is not None and d < D) else N.BC_TRANSMISSIVE
    cfg.pad = int(pad)
    cfg.dtype = {"f64": N.F64, "f32": N.F32, np.float64: N.F64, np.float32: N.F32}[dtype]
    cfg.layout = {"soa": N.SOA, "aos": N.AOS}[layout]
    cfg.kernel = {"fused": N.FUSED, "split": N.SPLIT}[kernel]
    cfg.gamma = float(gamma)
    cfg.nranks = int(nranks)
    cfg.rank = int(rank)
    cfg._nccl_keep = nccl_id  # keep the bytes alive
    cfg.nccl_id = ctypes.cast(ctypes.c_char_p(nccl_id), ctypes.c_void_p) if nccl_id else None
    cfg.device = int(device)
    cfg.stream = int(stream) if stream else None
    cfg.arena = int(arena) if arena else None
    cfg.rows_per_chunk = int(rows_per_chunk)
    cfg.transport = {"nccl": N.TRANSPORT_NCCL, "p2p": N.TRANSPORT_P2P,
                     "loopback": N.TRANSPORT_LOOPBACK,
                     "loopback_nccl": N.TRANSPORT_LOOPBACK_NCCL}[transport]
    cfg.order = int(order)
    return cfg


def halo_plan(**kw):
    """Host-only halo plan (rpl_halo_plan) as a list of dicts."""
    cfg = make_config(**kw)
    n = ctypes.c_int32(0)
    N.check(N.lib().rpl_halo_plan(ctypes.byref(cfg), None, 0, ctypes.byref(n)))
    arr = (N.HaloEdge * max(n.value, 1))()
    N.check(N.lib().rpl_halo_plan(ctypes.byref(cfg), arr, n.value, ctypes.byref(n)))
    out = []
    for e in arr[: n.value]:
        out.append(dict(src_part=e.src_part, dst_part=e.dst_part, src_lo=tuple(e.src_lo),
                        src_hi=tuple(e.src_hi), dst_lo=tuple(e.dst_lo), dst_hi=tuple(e.dst_hi),
                        mode=tuple(e.mode)))
    return out


def config_check(**kw):
    cfg = make_config(**kw)
    N.check(N.lib().rpl_config_check(ctypes.byref(cfg)))


def arena_bytes(**kw):
    cfg = make_config(**kw)
    out = ctypes.c_size_t(0)
    N.check(N.lib().rpl_arena_bytes(ctypes.byref(cfg), ctypes.byref(out)))
    return out.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    N.check(N.lib().rpl_nccl_unique_id(buf))
    return buf.raw


class Domain:
    """A padded, partitioned N-D tensor of Euler conserved states on one GPU (rank)."""

    def __init__(self, size, **kw):
        self.cfg = make_config(size, **kw)
        self.ndim = len(size)
        self.C = self.ndim + 2
        self.np_dtype = np.float64 if self.cfg.dtype == N.F64 else np.float32
        h = ctypes.c_void_p()
        N.check(N.lib().rpl_create(ctypes.byref(self.cfg), ctypes.byref(h)))
        self._h = h
        lo = (ctypes.c_int64 * 3)()
        hi = (ctypes.c_int64 * 3)()
        N.check(N.lib().rpl_local_box(self._h, lo, hi))
        self.lo = tuple(lo)
        self.hi = tuple(hi)
        self.box = tuple(hi[d] - lo[d] for d in range(3))

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None):
            N.lib().rpl_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- shapes
    def soa_shape(self):
        return (self.C,) + tuple(reversed(self.box[: self.ndim]))

    def aos_shape(self):
        return tuple(reversed(self.box[: self.ndim])) + (self.C,)

    # -- state
    def set_state(self, U: np.ndarray):
        """U: dense AoS interior of this rank's box, shape (nz, ny, nx, C)."""
        if U.shape != self.aos_shape():
            raise ValueError(f"shape {U.shape} != {self.aos_shape()}")
        soa = np.ascontiguousarray(np.moveaxis(U, -1, 0), dtype=self.np_dtype)
        N.check(N.lib().rpl_set_state(self._h, soa.ctypes.data))

    def get_state(self) -> np.ndarray:
        soa = np.empty(self.soa_shape(), dtype=self.np_dtype)
        N.check(N.lib().rpl_get_state(self._h, soa.ctypes.data))
        return np.ascontiguousarray(np.moveaxis(soa, 0, -1))

    def set_state_ptr(self, host_ptr: int):
        """Zero-copy: host_ptr -> dense SoA (C, nz, ny, nx) of the dtype (pinned for speed)."""
        N.check(N.lib().rpl_set_state(self._h, ctypes.c_void_p(host_ptr)))

    def get_state_ptr(self, host_ptr: int):
        N.check(N.lib().rpl_get_state(self._h, ctypes.c_void_p(host_ptr)))

    def get_padded(self, part: int = 0) -> np.ndarray:
        """Full padded buffer of a local partition, dense SoA (C, pz, py, px)."""
        p = self.cfg.pad
        ext = [(self.box[d] // self.cfg.parts[d] if self.cfg.nranks == 1 else self.box[d]) + 2 * p
               if d < self.ndim else 1 for d in range(3)]
        out = np.empty((self.C, ext[2], ext[1], ext[0]), dtype=self.np_dtype)
        N.check(N.lib().rpl_get_padded(self._h, int(part), out.ctypes.data))
        return out.reshape((self.C,) + tuple(reversed(ext[: self.ndim])))

    # -- the step
    def fill_padding(self):
        N.check(N.lib().rpl_fill_padding(self._h))

    def advance(self, dt: float, nsteps: int = 1):
        N.check(N.lib().rpl_advance(self._h, float(dt), int(nsteps)))

    def max_wavespeed(self) -> float:
        out = ctypes.c_double(0.0)
        N.check(N.lib().rpl_max_wavespeed(self._h, ctypes.byref(out)))
        return out.value

    def advance_cfl(self, t_end, cfl=0.9, n_reduced=5, reduce=0.2, max_steps=10_000_000):
        n = ctypes.c_int32(0)
        N.check(N.lib().rpl_advance_cfl(self._h, float(t_end), float(cfl), int(n_reduced),
                                        float(reduce), int(max_steps), ctypes.byref(n)))
        return n.value

    def advance_to(self, t_end, cfl=0.9, n_reduced=5, reduce=0.2, max_steps=10_000_000):
        """Device-side CFL run (rpl_advance_to).  Returns (t reached, steps taken)."""
        t = ctypes.c_double(0.0)
        n = ctypes.c_int32(0)
        N.check(N.lib().rpl_advance_to(self._h, float(t_end), float(cfl), int(n_reduced),
                                       float(reduce), int(max_steps), ctypes.byref(t),
                                       ctypes.byref(n)))
        return t.value, n.value

    def synchronize(self):
        N.check(N.lib().rpl_synchronize(self._h))

    # -- paper sec. 7.3 flux difference (Table 4 benchmark)
    def flux_difference(self, dt: float):
        N.check(N.lib().rpl_flux_difference(self._h, float(dt)))

    def get_flux_difference(self) -> np.ndarray:
        soa = np.empty(self.soa_shape(), dtype=self.np_dtype)
        N.check(N.lib().rpl_get_flux_difference(self._h, soa.ctypes.data))
        return np.ascontiguousarray(np.moveaxis(soa, 0, -1))

    # -- P2P transport (nranks > 1): export IPC blob, all-gather it, attach
    def p2p_export(self) -> bytes:
        n = ctypes.c_size_t(0)
        N.check(N.lib().rpl_p2p_export(self._h, None, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        N.check(N.lib().rpl_p2p_export(self._h, buf, ctypes.byref(n)))
        return buf.raw[: n.value]

    def p2p_attach(self, blobs):
        """blobs: list of every rank's export blob, in rank order."""
        size = len(blobs[0])
        assert all(len(b) == size for b in blobs)
        joined = b"".join(blobs)
        N.check(N.lib().rpl_p2p_attach(self._h, joined, size))

    def profile(self, max_launches: int):
        """Record CUDA events around every step-kernel launch (0 disables)."""
        N.check(N.lib().rpl_profile(self._h, int(max_launches)))

    def profile_read(self):
        """(summed kernel ms, launches) since the last read; synchronises."""
        ms = ctypes.c_double(0.0)
        n = ctypes.c_int64(0)
        N.check(N.lib().rpl_profile_read(self._h, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def profile_halo(self):
        """(summed exposed-halo ms, exchanges) since the last read (multi-rank; the
        interior-done -> halo-ready event pairs of rpl_profile_halo); synchronises."""
        ms = ctypes.c_double(0.0)
        n = ctypes.c_int64(0)
        N.check(N.lib().rpl_profile_halo(self._h, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def kernel_name(self, op: str = "step") -> str:
        """Name of the kernel rpl_advance ("step") or rpl_flux_difference
        ("fluxdiff") launches for this configuration."""
        return N.lib().rpl_kernel_name(self._h, {"step": 0, "fluxdiff": 1}[op]).decode()

    @property
    def launches_per_step(self) -> int:
        n = ctypes.c_int32(0)
        N.check(N.lib().rpl_launches_per_step(self._h, ctypes.byref(n)))
        return n.value
