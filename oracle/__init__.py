"""CPU oracle for the Ripple (arXiv 2104.08571) finite-volume step.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with the CUDA path (``paper_2104_08571_b200``,
``include/``); the two meet only through the seeded generators in
``workloads/`` (which hold none of the scheme's arithmetic).

The arithmetic lives in plain C (``ripple_oracle.c`` + ``oracle_scheme.inc``,
compiled with ``-O2 -ffp-contract=off``); this module only marshals numpy
arrays.  Every C function cites the passage it follows; the pins that tie it
to the paper and to mathematics are in ``tests/test_oracle_*.py``.

Parity status per function:
  step / sweep / fill_ghosts  -- pinned (P2-P8, linear-mode, acoustic, BC pins)
  max_wavespeed               -- pinned (closed-form states)
  riemann_exact               -- pinned (textbook star state, RH jump conditions)
  run_cfl                     -- pinned through P2 (Sod convergence)
  flux_difference             -- pinned (uniform state -> 0, Fourier symbol of the
                                 linear FORCE flux difference, 1-D sweep relation)
  step/sweep with order=2     -- pinned (limiter-inactive data == order 1 bitwise,
    (MUSCL-Hancock + FORCE)      L1 rate ~2 on a smooth wave, Sod bounds/convergence,
                                 conservation, symmetry, uniform state)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = [os.path.join(_HERE, "ripple_oracle.c")]
_DEPS = _SRC + [os.path.join(_HERE, "oracle_scheme.inc"), os.path.join(_HERE, "ripple_oracle.h")]
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

BC_TRANSMISSIVE, BC_PERIODIC, BC_REFLECTIVE = 0, 1, 2
OK, E_INVALID, E_DOMAIN = 0, -1, -7


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, no CUDA). Returns the .so path."""
    stale = force or not os.path.exists(_LIB_PATH) or any(
        os.path.getmtime(p) > os.path.getmtime(_LIB_PATH) for p in _DEPS)
    if stale:
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c11",
               "-o", tmp] + _SRC + ["-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class _Grid(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int), ("n", ctypes.c_long * 3), ("pad", ctypes.c_int),
                ("dx", ctypes.c_double * 3), ("gamma", ctypes.c_double),
                ("bc_lo", ctypes.c_int * 3), ("bc_hi", ctypes.c_int * 3),
                ("order", ctypes.c_int)]


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        dp, fp = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_float)
        gp = ctypes.POINTER(_Grid)
        _lib.orc_step_f64.argtypes = [gp, dp, ctypes.c_double, ctypes.c_int]
        _lib.orc_step_f32.argtypes = [gp, fp, ctypes.c_double, ctypes.c_int]
        _lib.orc_sweep_f64.argtypes = [gp, dp, ctypes.c_double, ctypes.c_int]
        _lib.orc_fill_ghosts_f64.argtypes = [gp, dp]
        _lib.orc_fill_ghosts_f64.restype = None
        _lib.orc_max_wavespeed_f64.argtypes = [gp, dp]
        _lib.orc_max_wavespeed_f64.restype = ctypes.c_double
        _lib.orc_max_wavespeed_f32.argtypes = [gp, fp]
        _lib.orc_max_wavespeed_f32.restype = ctypes.c_double
        _lib.orc_run_cfl_f64.argtypes = [gp, dp, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                         ctypes.c_double, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_int)]
        _lib.orc_flux_difference_f64.argtypes = [gp, dp, ctypes.c_double, dp]
        _lib.orc_flux_difference_f32.argtypes = [gp, fp, ctypes.c_double, fp]
        _lib.orc_riemann_exact.argtypes = [ctypes.c_double] * 7 + [dp, ctypes.c_long, dp, dp]
        _lib.orc_set_threads.argtypes = [ctypes.c_int]
        _lib.orc_set_threads.restype = ctypes.c_int
        _lib.orc_set_threads(1)  # single-threaded unless set_threads() asks for more
    return _lib


class Grid:
    """Geometry + scheme constants (SURVEY 8(c) input line)."""

    def __init__(self, n, pad=2, dx=None, gamma=1.4, bc_lo=None, bc_hi=None, order=1):
        n = tuple(int(v) for v in n)
        self.ndim = len(n)
        assert 1 <= self.ndim <= 3
        self.n = n
        self.pad = int(pad)
        self.dx = tuple(float(v) for v in (dx if dx is not None else [1.0 / v for v in n]))
        self.gamma = float(gamma)
        self.bc_lo = tuple(bc_lo if bc_lo is not None else [BC_TRANSMISSIVE] * self.ndim)
        self.bc_hi = tuple(bc_hi if bc_hi is not None else [BC_TRANSMISSIVE] * self.ndim)
        self.order = int(order)

    @property
    def C(self):
        return self.ndim + 2

    def shape(self):
        """numpy shape of the dense AoS interior array: (nz, ny, nx, C) trimmed to ndim."""
        return tuple(reversed(self.n)) + (self.C,)

    def _c(self):
        g = _Grid()
        g.ndim = self.ndim
        for d in range(3):
            g.n[d] = self.n[d] if d < self.ndim else 1
            g.dx[d] = self.dx[d] if d < self.ndim else 1.0
            g.bc_lo[d] = self.bc_lo[d] if d < self.ndim else 0
            g.bc_hi[d] = self.bc_hi[d] if d < self.ndim else 0
        g.pad = self.pad
        g.gamma = self.gamma
        g.order = self.order
        return g


class DomainError(RuntimeError):
    pass


def set_threads(n: int) -> int:
    """OpenMP threads of the oracle's line loops (step, sweep, flux_difference);
    default 1.  Lines are independent: results are bitwise the same for any count."""
    return int(_L().orc_set_threads(int(n)))


def _check(rc):
    if rc == E_DOMAIN:
        raise DomainError("oracle: rho<=0, p<=0 or non-finite state (S:588)")
    if rc != OK:
        raise ValueError(f"oracle: invalid argument (rc={rc})")


def _arr(U, dtype):
    if U.dtype != dtype or not U.flags.c_contiguous:
        raise TypeError(f"expected C-contiguous {dtype}")
    return U.ctypes.data_as(ctypes.POINTER(ctypes.c_double if dtype == np.float64
                                           else ctypes.c_float))


def step(grid: Grid, U: np.ndarray, dt: float, nsteps: int = 1) -> np.ndarray:
    """Return U after nsteps split FORCE steps (Listing 8). Copies U."""
    U = np.ascontiguousarray(U).copy()
    g = grid._c()
    if U.dtype == np.float64:
        _check(_L().orc_step_f64(ctypes.byref(g), _arr(U, np.float64), float(dt), int(nsteps)))
    elif U.dtype == np.float32:
        _check(_L().orc_step_f32(ctypes.byref(g), _arr(U, np.float32), float(dt), int(nsteps)))
    else:
        raise TypeError(U.dtype)
    return U


def sweep(grid: Grid, U: np.ndarray, dt: float, d: int) -> np.ndarray:
    """One sweep along direction d (fp64): ghost fill + FORCE faces + update."""
    U = np.ascontiguousarray(U, dtype=np.float64).copy()
    _check(_L().orc_sweep_f64(ctypes.byref(grid._c()), _arr(U, np.float64), float(dt), int(d)))
    return U


def padded_shape(grid: Grid):
    return tuple(v + 2 * grid.pad for v in reversed(grid.n)) + (grid.C,)


def fill_ghosts(grid: Grid, P: np.ndarray) -> np.ndarray:
    """Fill the ghost layers of a padded fp64 AoS array. Copies P."""
    P = np.ascontiguousarray(P, dtype=np.float64).copy()
    assert P.shape == padded_shape(grid)
    _L().orc_fill_ghosts_f64(ctypes.byref(grid._c()), _arr(P, np.float64))
    return P


def flux_difference(grid: Grid, U: np.ndarray, dt: float) -> np.ndarray:
    """R = sum_d (F_{i+1/2} - F_{i-1/2}) with FORCE (paper sec. 7.3, Table 4 kernel)."""
    U = np.ascontiguousarray(U)
    R = np.empty_like(U)
    g = grid._c()
    if U.dtype == np.float64:
        _check(_L().orc_flux_difference_f64(ctypes.byref(g), _arr(U, np.float64), float(dt),
                                            _arr(R, np.float64)))
    else:
        _check(_L().orc_flux_difference_f32(ctypes.byref(g), _arr(U, np.float32), float(dt),
                                            _arr(R, np.float32)))
    return R


def max_wavespeed(grid: Grid, U: np.ndarray) -> float:
    """max over cells of |u| + c."""
    U = np.ascontiguousarray(U)
    g = grid._c()
    if U.dtype == np.float64:
        return _L().orc_max_wavespeed_f64(ctypes.byref(g), _arr(U, np.float64))
    return _L().orc_max_wavespeed_f32(ctypes.byref(g), _arr(U, np.float32))


def run_cfl(grid: Grid, U: np.ndarray, t_end: float, cfl: float = 0.9, n_reduced: int = 5,
            reduce: float = 0.2, max_steps: int = 10_000_000):
    """CFL-driven run to t_end (Listing 8 wavespeed -> max -> dt; readings D3, S8).
    Returns (U, nsteps)."""
    U = np.ascontiguousarray(U, dtype=np.float64).copy()
    n = ctypes.c_int(0)
    _check(_L().orc_run_cfl_f64(ctypes.byref(grid._c()), _arr(U, np.float64), float(t_end),
                                float(cfl), int(n_reduced), float(reduce), int(max_steps),
                                ctypes.byref(n)))
    return U, n.value


def riemann_exact(left, right, gamma, xi):
    """Exact 1-D Riemann solution (Toro ch. 4). left/right = (rho, u, p).
    Returns (star=(p*, u*, rho*L, rho*R), W[len(xi), 3] primitive samples)."""
    xi = np.ascontiguousarray(xi, dtype=np.float64)
    out = np.zeros((len(xi), 3))
    star = np.zeros(4)
    it = _L().orc_riemann_exact(*[float(v) for v in left], *[float(v) for v in right],
                                float(gamma), _arr(xi, np.float64), len(xi),
                                _arr(star, np.float64), _arr(out, np.float64))
    if it < 0:
        raise ValueError("vacuum generated")
    return tuple(star), out
