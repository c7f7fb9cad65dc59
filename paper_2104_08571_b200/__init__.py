"""B200-native hot path of Ripple (arXiv 2104.08571): the split FORCE finite-volume step.

Product path: libripple_fv.so (hand-written sm_100a CUDA kernels behind the
C ABI of include/ripple_fv.h) + this thin ctypes binding.  No CPU fallback.
"""
from ._native import (AOS, BC_PERIODIC, BC_REFLECTIVE, BC_TRANSMISSIVE, F32, F64, FUSED,  # noqa
                      MAP_BROADCAST, MAP_REFLECT, MAP_TRANSLATE, SOA, SPLIT, DomainError,
                      RplError, lib)
from .domain import (Domain, arena_bytes, config_check, halo_plan, make_config,  # noqa
                     nccl_unique_id)

__all__ = ["Domain", "halo_plan", "make_config", "config_check", "arena_bytes",
           "nccl_unique_id", "DomainError", "RplError", "lib"]
