"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the scheme (no flux, no update, no boundary
rule): it only defines initial data.  Every field is a pure function of
(seed, global cell index), so any partitioning of the grid sees the same
values (SURVEY 8(d) "Concrete synthetic inputs").

Arrays are dense AoS interiors, shape (nz, ny, nx, C) trimmed to ndim, with
conserved components [rho, m_x, (m_y), (m_z), E] (SURVEY reading S6).  The
primitive -> conserved map used to *define* the initial data is
E = p/(gamma-1) + 1/2 rho |u|^2.
"""
from __future__ import annotations

import math

import numpy as np

SEED = 20210418
GAMMA = 1.4

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (stateless, counter-based)."""
    with np.errstate(over="ignore"):
        z = (x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def uniform_pm1(seed: int, stream: int, index: np.ndarray) -> np.ndarray:
    """U[-1, 1) from splitmix64(seed ^ (index * 8 + stream))."""
    key = (index.astype(np.uint64) * np.uint64(8) + np.uint64(stream)) ^ np.uint64(seed)
    z = splitmix64(key)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -52) - 1.0


def _box(n, box):
    D = len(n)
    if box is None:
        return [0] * D, list(n)
    lo, hi = box
    return [int(v) for v in lo[:D]], [int(v) for v in hi[:D]]


def _global_index(n, box=None):
    """Global linear cell index (x fastest) of the cells of `box` (default: the whole
    grid), shape (nz, ny, nx) trimmed to ndim."""
    D = len(n)
    lo, hi = _box(n, box)
    axes = [np.arange(lo[d], hi[d], dtype=np.uint64) for d in range(D)]
    stride = [int(np.prod(n[:d])) for d in range(D)]
    mesh = np.meshgrid(*reversed(axes), indexing="ij")
    idx = np.zeros(mesh[0].shape, dtype=np.uint64)
    for d in range(D):
        idx += mesh[D - 1 - d] * np.uint64(stride[d])
    return idx


def _coords(n, dx, origin=None, box=None):
    """Cell-centre coordinates x_d = (i_d + 1/2) dx_d of the cells of `box`."""
    D = len(n)
    origin = origin or [0.0] * D
    lo, hi = _box(n, box)
    axes = [origin[d] + (np.arange(lo[d], hi[d]) + 0.5) * dx[d] for d in range(D)]
    mesh = np.meshgrid(*reversed(axes), indexing="ij")  # (z, y, x) order
    return list(reversed(mesh))  # [x, y, z]


def conserved(rho, vel, p, gamma=GAMMA):
    """Stack (rho, u_vec, p) into conserved [rho, rho*u_k..., E]."""
    D = len(vel)
    ke = 0.5 * rho * sum(v * v for v in vel)
    E = p / (gamma - 1.0) + ke
    comps = [rho] + [rho * v for v in vel] + [E]
    return np.stack(comps, axis=-1).astype(np.float64)


def uniform(n, rho=1.0, vel=None, p=1.0, gamma=GAMMA):
    D = len(n)
    vel = vel if vel is not None else [0.0] * D
    shape = tuple(reversed(n))
    return conserved(np.full(shape, rho), [np.full(shape, v) for v in vel], np.full(shape, p),
                     gamma)


def random_state(n, seed=SEED, gamma=GAMMA, rho=(0.5, 1.5), vel=0.5, p=(0.5, 1.5), box=None):
    """Random positive state: rho, p uniform in the given ranges, |u_k| <= vel.
    `box` = (lo, hi) restricts generation to a sub-box of the global grid."""
    D = len(n)
    idx = _global_index(n, box)
    r = rho[0] + (rho[1] - rho[0]) * 0.5 * (uniform_pm1(seed, 0, idx) + 1.0)
    vs = [vel * uniform_pm1(seed, 1 + k, idx) for k in range(D)]
    pr = p[0] + (p[1] - p[0]) * 0.5 * (uniform_pm1(seed, 4, idx) + 1.0)
    return conserved(r, vs, pr, gamma)


def sod(n=200, x0=0.5, gamma=GAMMA, left=(1.0, 0.0, 1.0), right=(0.125, 0.0, 0.1)):
    """Sod (1978) shock tube on [0,1]: cell i is left iff x_i < x0 (reading S12)."""
    x = (np.arange(n) + 0.5) / n
    L = x < x0
    rho = np.where(L, left[0], right[0])
    u = np.where(L, left[1], right[1])
    p = np.where(L, left[2], right[2])
    return conserved(rho, [u], p, gamma)


def sod_embedded(n, axis, gamma=GAMMA, mirrored=False):
    """1-D Sod along `axis` of an N-D grid (SURVEY pin P7); other axes uniform."""
    D = len(n)
    N = n[axis]
    x = (np.arange(N) + 0.5) / N
    L = x < 0.5
    if mirrored:
        L = ~L
    shape = tuple(reversed(n))
    bshape = [1] * D
    bshape[D - 1 - axis] = N
    rho = np.broadcast_to(np.where(L, 1.0, 0.125).reshape(bshape), shape)
    p = np.broadcast_to(np.where(L, 1.0, 0.1).reshape(bshape), shape)
    vel = [np.zeros(shape) for _ in range(D)]
    return conserved(np.array(rho), vel, np.array(p), gamma)


def smooth_density_wave(n, vel, amp=0.2, k=None, rho0=1.0, p0=1.0, gamma=GAMMA):
    """rho = rho0 + amp*sin(2 pi k.x) with uniform velocity and pressure on [0,1]^D
    (a contact/entropy wave: exact solution is a translation, SURVEY pin P3)."""
    D = len(n)
    k = k if k is not None else [1] * D
    X = _coords(n, [1.0 / v for v in n])
    phase = sum(2.0 * math.pi * k[d] * X[d] for d in range(D))
    rho = rho0 + amp * np.sin(phase)
    shape = rho.shape
    return conserved(rho, [np.full(shape, float(v)) for v in vel], np.full(shape, p0), gamma)


def mach_shock_state(mach=3.81, pre=(1.0, 0.0, 1.0), gamma=GAMMA):
    """Post-shock primitive state of a normal shock of Mach `mach` moving into `pre`
    (Rankine-Hugoniot; SURVEY reading S22 / Appendix B)."""
    r1, u1, p1 = pre
    c1 = math.sqrt(gamma * p1 / r1)
    M2 = mach * mach
    r2 = r1 * (gamma + 1.0) * M2 / ((gamma - 1.0) * M2 + 2.0)
    p2 = p1 * (2.0 * gamma * M2 - (gamma - 1.0)) / (gamma + 1.0)
    S = u1 + mach * c1
    u2 = S * (1.0 - r1 / r2) + u1 * r1 / r2
    return r2, u2, p2


def shock_bubble(n, dx=None, seed=SEED, gamma=GAMMA, shock_x=0.1, radius=0.15,
                 bubble_rho=0.1, perturb=1e-3, origin=None, box=None):
    """Mach 3.81 shock hitting a light bubble (the paper's scaling workload, P:1369-1373,
    geometry of SURVEY 8(d)): post-shock state for x < shock_x, quiescent (1,0,1)
    elsewhere, bubble of density bubble_rho centred at (0.4, L_y/2, L_z/2), and
    rho *= (1 + perturb * xi) with xi ~ U[-1,1) from the hash generator."""
    D = len(n)
    dx = dx if dx is not None else [1.0 / n[0]] * D
    X = _coords(n, dx, origin, box)
    L = [n[d] * dx[d] for d in range(D)]
    r2, u2, p2 = mach_shock_state(3.81, (1.0, 0.0, 1.0), gamma)
    post = X[0] < shock_x
    centre = [0.4] + [0.5 * L[d] for d in range(1, D)]
    dist2 = sum((X[d] - centre[d]) ** 2 for d in range(D))
    bubble = (dist2 < radius * radius) & ~post
    rho = np.where(post, r2, np.where(bubble, bubble_rho, 1.0))
    u = np.where(post, u2, 0.0)
    p = np.where(post, p2, 1.0)
    xi = uniform_pm1(seed, 5, _global_index(n, box))
    rho = rho * (1.0 + perturb * xi)
    vel = [u] + [np.zeros_like(u) for _ in range(1, D)]
    return conserved(rho, vel, p, gamma)


# BASELINE.json configs -> (ndim, global size, pad, dtype, steps); names used by bench/tests.
CONFIGS = {
    "sod": dict(ndim=1, n=(200,), pad=2, dtype="f64", t_end=0.2),
    "2d1024": dict(ndim=2, n=(1024, 1024), pad=2, dtype="f64", steps=100),
    "s512": dict(ndim=3, n=(512, 512, 512), pad=2, dtype="f64", steps=100),
    "w384": dict(ndim=3, n=(384, 384, 384), pad=2, dtype="f32", steps=100),
    "l256": dict(ndim=3, n=(256, 256, 256), pad=2, dtype="f32", steps=100),
}

S0_SHOCK_BUBBLE = None  # computed at run time by each side's max_wavespeed


def fixed_dt(S0, dx_min, cfl=0.4):
    """Fixed dt recipe of SURVEY 8(d): dt = 0.4 min dx / S0 (input parameter, not scheme)."""
    return cfl * dx_min / S0
