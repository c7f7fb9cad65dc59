"""ctypes declarations of include/ripple_fv.h (argument marshalling only).

Loading fails loudly if the native library is missing: there is no Python or
CPU fallback for any operation of the step.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# RPL_LIB: another build of the library (A/B comparisons of kernel forms on one box)
LIB_PATH = os.environ.get("RPL_LIB") or os.path.join(HERE, "libripple_fv.so")

RPL_OK = 0
STATUS = {0: "RPL_OK", -1: "RPL_E_INVALID_ARG", -2: "RPL_E_NOT_DIVISIBLE",
          -3: "RPL_E_PAD_TOO_SMALL", -4: "RPL_E_OOM", -5: "RPL_E_CUDA", -6: "RPL_E_NCCL",
          -7: "RPL_E_DOMAIN", -8: "RPL_E_SHAPE_MISMATCH", -9: "RPL_E_UNSUPPORTED"}
F32, F64 = 0, 1
SOA, AOS = 0, 1
FUSED, SPLIT = 0, 1
TRANSPORT_NCCL, TRANSPORT_P2P, TRANSPORT_LOOPBACK, TRANSPORT_LOOPBACK_NCCL = 0, 1, 2, 3
BC_TRANSMISSIVE, BC_PERIODIC, BC_REFLECTIVE = 0, 1, 2
MAP_TRANSLATE, MAP_REFLECT, MAP_BROADCAST = 0, 1, 2


class Config(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int32), ("size", ctypes.c_int64 * 3), ("pad", ctypes.c_int32),
                ("parts", ctypes.c_int32 * 3), ("dtype", ctypes.c_int), ("layout", ctypes.c_int),
                ("kernel", ctypes.c_int), ("gamma", ctypes.c_double), ("dx", ctypes.c_double * 3),
                ("bc_lo", ctypes.c_int * 3), ("bc_hi", ctypes.c_int * 3),
                ("nranks", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("nccl_id", ctypes.c_void_p), ("device", ctypes.c_int32),
                ("stream", ctypes.c_void_p), ("arena", ctypes.c_void_p),
                ("rows_per_chunk", ctypes.c_int32), ("transport", ctypes.c_int),
                ("order", ctypes.c_int32)]


class HaloEdge(ctypes.Structure):
    _fields_ = [("src_part", ctypes.c_int32), ("dst_part", ctypes.c_int32),
                ("src_lo", ctypes.c_int64 * 3), ("src_hi", ctypes.c_int64 * 3),
                ("dst_lo", ctypes.c_int64 * 3), ("dst_hi", ctypes.c_int64 * 3),
                ("mode", ctypes.c_int32 * 3)]


EXPORTS = ["rpl_config_init", "rpl_config_check", "rpl_arena_bytes", "rpl_nccl_unique_id",
           "rpl_create", "rpl_local_box", "rpl_set_state", "rpl_get_state", "rpl_get_padded",
           "rpl_fill_padding", "rpl_advance", "rpl_max_wavespeed", "rpl_advance_cfl",
           "rpl_advance_to",
           "rpl_synchronize", "rpl_launches_per_step", "rpl_profile", "rpl_profile_read",
           "rpl_profile_halo", "rpl_kernel_name",
           "rpl_halo_plan", "rpl_p2p_export", "rpl_p2p_attach",
           "rpl_flux_difference", "rpl_get_flux_difference", "rpl_destroy",
           "rpl_last_error"]

_lib = None


def lib():
    """Load libripple_fv.so (built by __graft_entry__.build() / _build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"native library missing: {LIB_PATH} -- run python -c "
                          "'import __graft_entry__ as g; g.build()' (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    P = ctypes.POINTER
    vp, st = ctypes.c_void_p, ctypes.c_int
    L.rpl_config_init.argtypes = [P(Config)]
    L.rpl_config_init.restype = None
    L.rpl_config_check.argtypes = [P(Config)]
    L.rpl_arena_bytes.argtypes = [P(Config), P(ctypes.c_size_t)]
    L.rpl_nccl_unique_id.argtypes = [vp]
    L.rpl_create.argtypes = [P(Config), P(vp)]
    L.rpl_local_box.argtypes = [vp, P(ctypes.c_int64), P(ctypes.c_int64)]
    L.rpl_set_state.argtypes = [vp, vp]
    L.rpl_get_state.argtypes = [vp, vp]
    L.rpl_get_padded.argtypes = [vp, ctypes.c_int32, vp]
    L.rpl_fill_padding.argtypes = [vp]
    L.rpl_advance.argtypes = [vp, ctypes.c_double, ctypes.c_int32]
    L.rpl_max_wavespeed.argtypes = [vp, P(ctypes.c_double)]
    L.rpl_advance_cfl.argtypes = [vp, ctypes.c_double, ctypes.c_double, ctypes.c_int32,
                                  ctypes.c_double, ctypes.c_int32, P(ctypes.c_int32)]
    L.rpl_advance_to.argtypes = [vp, ctypes.c_double, ctypes.c_double, ctypes.c_int32,
                                 ctypes.c_double, ctypes.c_int32, P(ctypes.c_double),
                                 P(ctypes.c_int32)]
    L.rpl_synchronize.argtypes = [vp]
    L.rpl_launches_per_step.argtypes = [vp, P(ctypes.c_int32)]
    L.rpl_profile.argtypes = [vp, ctypes.c_int32]
    L.rpl_profile_read.argtypes = [vp, P(ctypes.c_double), P(ctypes.c_int64)]
    L.rpl_profile_halo.argtypes = [vp, P(ctypes.c_double), P(ctypes.c_int64)]
    L.rpl_kernel_name.argtypes = [vp, ctypes.c_int32]
    L.rpl_kernel_name.restype = ctypes.c_char_p
    L.rpl_halo_plan.argtypes = [P(Config), P(HaloEdge), ctypes.c_int32, P(ctypes.c_int32)]
    L.rpl_p2p_export.argtypes = [vp, vp, P(ctypes.c_size_t)]
    L.rpl_p2p_attach.argtypes = [vp, vp, ctypes.c_size_t]
    L.rpl_flux_difference.argtypes = [vp, ctypes.c_double]
    L.rpl_get_flux_difference.argtypes = [vp, vp]
    L.rpl_destroy.argtypes = [vp]
    L.rpl_destroy.restype = None
    L.rpl_last_error.argtypes = []
    L.rpl_last_error.restype = ctypes.c_char_p
    for name in EXPORTS:
        if name not in ("rpl_config_init", "rpl_destroy", "rpl_last_error", "rpl_kernel_name"):
            getattr(L, name).restype = st
    _lib = L
    return L


class RplError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class DomainError(RplError):
    """rho <= 0, p <= 0 or non-finite state."""


def check(status):
    if status != RPL_OK:
        msg = lib().rpl_last_error().decode(errors="replace")
        if status == -7:
            raise DomainError(status, msg)
        raise RplError(status, msg)
