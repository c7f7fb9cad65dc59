"""Order-2 reconstruction (MUSCL-Hancock + FORCE = Toro's SLIC, minmod
slopes; readings F3a-F3d) on the GPU against the order-2 oracle.

Same bar as order 1 (BASELINE.json north_star): max relative error <= 1e-10 in
fp64, <= 1e-4 in fp32, metric of DESIGN.md reading S15; fused vs split kernels,
AoS vs SoA and any partitioning bitwise identical.
"""
import numpy as np
import pytest

import oracle
import paper_2104_08571_b200 as R
import workloads as W
from test_parity_gpu import OK, relerr

pytestmark = pytest.mark.gpu


def gpu(U0, dt, nsteps, dtype="f64", **kw):
    n = tuple(reversed(U0.shape[:-1]))
    with R.Domain(n, dtype=dtype, order=2, **kw) as dom:
        dom.set_state(U0)
        dom.advance(dt, nsteps)
        return dom.get_state()


def orc(U0, dt, nsteps, dx, bc_lo=None, bc_hi=None):
    n = tuple(reversed(U0.shape[:-1]))
    D = len(n)
    g = oracle.Grid(n, pad=2, dx=dx, order=2,
                    bc_lo=[OK[b] for b in (bc_lo or ["clamp"] * D)],
                    bc_hi=[OK[b] for b in (bc_hi or ["clamp"] * D)])
    return oracle.step(g, U0, dt, nsteps)


def test_sod_order2_cfl_matches_oracle():
    N = 200
    U0 = W.sod(N)
    with R.Domain((N,), pad=2, order=2) as dom:
        dom.set_state(U0)
        n = dom.advance_cfl(0.2)
        Ug = dom.get_state()
    Uo, no = oracle.run_cfl(oracle.Grid((N,), pad=2, order=2), U0, 0.2)
    assert n == no
    assert relerr(Ug, Uo) <= 1e-10


@pytest.mark.parametrize("kernel", ["fused", "split"])
@pytest.mark.parametrize("n", [(130, 70), (61, 45)])
def test_2d_order2_matches_oracle(kernel, n):
    dx = [1.0 / n[0]] * 2
    U0 = W.shock_bubble(n, dx=dx)
    dt = 0.4 * dx[0] / oracle.max_wavespeed(oracle.Grid(n), U0)
    assert relerr(gpu(U0, dt, 60, kernel=kernel, dx=dx), orc(U0, dt, 60, dx)) <= 1e-10


@pytest.mark.parametrize("bc", ["periodic", "reflective"])
def test_2d_order2_boundary_kinds(bc):
    n = (96, 50)
    dx = [1.0 / 96] * 2
    U0 = W.random_state(n, seed=4)
    dt = 0.3 * dx[0] / oracle.max_wavespeed(oracle.Grid(n), U0)
    kw = dict(bc_lo=[bc, bc], bc_hi=[bc, bc])
    assert relerr(gpu(U0, dt, 40, dx=dx, **kw), orc(U0, dt, 40, dx, **kw)) <= 1e-10


def test_3d_order2_matches_oracle():
    n = (24, 20, 16)
    dx = [1.0 / 24] * 3
    U0 = W.shock_bubble(n, dx=dx)
    dt = 0.4 * dx[0] / oracle.max_wavespeed(oracle.Grid(n), U0)
    assert relerr(gpu(U0, dt, 30, dx=dx), orc(U0, dt, 30, dx)) <= 1e-10


@pytest.mark.parametrize("n", [(128, 96), (24, 20, 16)])
def test_order2_fp32_against_fp32_oracle(n):
    D = len(n)
    dx = [1.0 / n[0]] * D
    U0 = W.shock_bubble(n, dx=dx).astype(np.float32)
    dt = 0.4 * dx[0] / oracle.max_wavespeed(oracle.Grid(n), U0.astype(np.float64))
    Uo = orc(U0, dt, 50, dx)
    assert Uo.dtype == np.float32
    assert relerr(gpu(U0, dt, 50, dtype="f32", dx=dx), Uo) <= 1e-4


@pytest.mark.parametrize("n,parts", [((130, 70), (2, 2)), ((130, 70), (1, 5)),
                                     ((24, 20, 16), (2, 1, 2)), ((200,), (4,))])
@pytest.mark.parametrize("bc", ["clamp", "periodic", "reflective"])
def test_order2_kernels_partitions_layouts_bitwise(n, parts, bc):
    D = len(n)
    dx = [1.0 / n[0]] * D
    U0 = W.random_state(n, seed=21)
    dt = 0.25 * dx[0] / 3.0
    kw = dict(dx=dx, bc_lo=[bc] * D, bc_hi=[bc] * D)
    ref = gpu(U0, dt, 12, **kw)
    for extra in [dict(kernel="split"), dict(parts=parts), dict(parts=parts, kernel="split"),
                  dict(layout="aos", kernel="split")]:
        assert np.array_equal(gpu(U0, dt, 12, **kw, **extra), ref), extra


def test_order2_device_cfl_matches_oracle():
    n = (130, 70)
    dx = [1.0 / 130] * 2
    U0 = W.shock_bubble(n, dx=dx)
    with R.Domain(n, dx=dx, order=2) as dom:
        dom.set_state(U0)
        t, steps = dom.advance_to(0.03)
        Ug = dom.get_state()
    Uo, no = oracle.run_cfl(oracle.Grid(n, dx=dx, order=2), U0, 0.03)
    assert steps == no and t == 0.03
    assert relerr(Ug, Uo) <= 1e-10


def test_order2_is_more_accurate_on_smooth_data():
    """Sanity on the device: the smooth-wave L1 error of order 2 is far below order 1."""
    N = 256
    per = ["periodic"]
    U0 = W.smooth_density_wave((N,), vel=[1.0])
    nst = int(np.ceil(0.25 / (0.5 / N / 2.2)))
    dt = 0.25 / nst
    errs = []
    for order in (1, 2):
        with R.Domain((N,), order=order, bc_lo=per, bc_hi=per) as dom:
            dom.set_state(U0)
            dom.advance(dt, nst)
            U = dom.get_state()
        shift = N // 4   # u t = 1/4 of the period (exact translation)
        errs.append(np.abs(U[:, 0] - np.roll(U0[:, 0], shift)).mean())
    assert errs[1] < 0.2 * errs[0], errs


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_order2_2d_fused_bitwise(dtype):
    """The 2-D order-2 fused kernel gives the split kernel's bit pattern (ragged
    windows and tiles, mixed boundaries)."""
    from test_parity_gpu import bits_equal
    n = (130, 61)
    dx = [1.0 / 130] * 2
    U0 = W.shock_bubble(n, dx=dx)
    if dtype == "f32":
        U0 = U0.astype(np.float32)
    dt = 0.4 * dx[0] / 5.8
    kw = dict(dx=dx, bc_lo=["reflective", "periodic"], bc_hi=["clamp", "periodic"])
    ref = gpu(U0, dt, 6, dtype=dtype, kernel="split", **kw)
    assert bits_equal(gpu(U0, dt, 6, dtype=dtype, **kw), ref)
