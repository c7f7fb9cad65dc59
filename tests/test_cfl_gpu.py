"""Device-side CFL step (`rpl_advance_to`) against the CPU oracle.

The oracle's `run_cfl` follows Listing 8's set_wavespeeds -> reduce(Max) ->
set_dt loop with the IEEE |u| + c formula; the device run derives
S from the step kernels' in-kernel wavespeeds (MUFU rsqrt/rcp + Newton, DESIGN.md
reading "device CFL"), so dt may differ in the last bits: the step count must
match exactly and the state within the north_star tolerance.  Between kernels
(split / fused, any partitioning) the device run is bitwise identical, because
every kernel evaluates the same per-cell wavespeed and max is exact.
"""
import numpy as np
import pytest

import oracle
import paper_2104_08571_b200 as R
import workloads as W
from test_parity_gpu import relerr

pytestmark = pytest.mark.gpu


def device_run(U0, t_end, dtype="f64", max_steps=10_000_000, **kw):
    n = tuple(reversed(U0.shape[:-1]))
    with R.Domain(n, dtype=dtype, **kw) as dom:
        dom.set_state(U0)
        t, steps = dom.advance_to(t_end, cfl=0.9, n_reduced=5, reduce=0.2, max_steps=max_steps)
        return dom.get_state(), t, steps


def host_run(U0, t_end, dtype="f64", **kw):
    n = tuple(reversed(U0.shape[:-1]))
    with R.Domain(n, dtype=dtype, **kw) as dom:
        dom.set_state(U0)
        steps = dom.advance_cfl(t_end, cfl=0.9, n_reduced=5, reduce=0.2)
        return dom.get_state(), steps


@pytest.mark.parametrize("kernel", ["split", "fused"])
def test_sod_device_cfl_matches_oracle(kernel):
    N = 200
    U0 = W.sod(N)
    Ug, t, n = device_run(U0, 0.2, pad=2, kernel=kernel)
    Uo, no = oracle.run_cfl(oracle.Grid((N,), pad=2), U0, 0.2)
    assert n == no == 100
    assert t == 0.2
    assert relerr(Ug, Uo) <= 1e-10


@pytest.mark.parametrize("n,t_end", [((130, 70), 0.04), ((20, 18, 16), 0.06)])
def test_shock_bubble_device_cfl_matches_oracle(n, t_end):
    D = len(n)
    dx = [1.0 / n[0]] * D
    U0 = W.shock_bubble(n, dx=dx)
    Ug, t, steps = device_run(U0, t_end, dx=dx)
    g = oracle.Grid(n, dx=dx)
    Uo, no = oracle.run_cfl(g, U0, t_end)
    assert steps == no and steps > 10
    assert t == t_end
    assert relerr(Ug, Uo) <= 1e-10


def test_device_cfl_matches_host_loop():
    n = (192, 160)
    dx = [1.0 / 192] * 2
    U0 = W.shock_bubble(n, dx=dx)
    Ud, t, nd = device_run(U0, 0.05, dx=dx)
    Uh, nh = host_run(U0, 0.05, dx=dx)
    assert nd == nh
    assert relerr(Ud, Uh) <= 1e-12


@pytest.mark.parametrize("n,parts", [((130, 70), (2, 2)), ((130, 70), (1, 5)),
                                     ((20, 18, 16), (1, 2, 2))])
def test_device_cfl_bitwise_across_kernels_and_partitions(n, parts):
    D = len(n)
    dx = [1.0 / n[0]] * D
    U0 = W.shock_bubble(n, dx=dx)
    ref, t0, n0 = device_run(U0, 0.03, dx=dx)
    for kw in [dict(kernel="split"), dict(parts=parts), dict(parts=parts, kernel="split")]:
        U, t, steps = device_run(U0, 0.03, dx=dx, **kw)
        assert steps == n0 and t == t0
        assert np.array_equal(U, ref), kw


@pytest.mark.parametrize("chunk", ["1", "3", "64"])
def test_device_cfl_chunking_is_invisible(chunk, monkeypatch):
    """Launches past t_end (chunk overshoot) must be skipped: any chunk size gives
    the same steps, time and bitwise state."""
    n = (96, 64)
    dx = [1.0 / 96] * 2
    U0 = W.shock_bubble(n, dx=dx)
    ref = device_run(U0, 0.02, dx=dx)
    monkeypatch.setenv("RPL_CFL_CHUNK", chunk)
    for kw in [{}, dict(kernel="split")]:
        got = device_run(U0, 0.02, dx=dx, **kw)
        assert got[1] == ref[1] and got[2] == ref[2]
        assert np.array_equal(got[0], ref[0])


def test_device_cfl_fp32():
    n = (128, 96)
    dx = [1.0 / 128] * 2
    U0 = W.shock_bubble(n, dx=dx)
    Ug, t, steps = device_run(U0.astype(np.float32), 0.03, dtype="f32", dx=dx)
    Uo, no = oracle.run_cfl(oracle.Grid(n, dx=dx), U0, 0.03)
    assert steps == no
    assert relerr(Ug, Uo) <= 1e-4


def test_device_cfl_max_steps_and_zero_time():
    n = (96, 64)
    dx = [1.0 / 96] * 2
    U0 = W.shock_bubble(n, dx=dx)
    U7, t7, n7 = device_run(U0, 1.0, max_steps=7, dx=dx)
    assert n7 == 7 and 0.0 < t7 < 1.0
    Uo, no = oracle.run_cfl(oracle.Grid(n, dx=dx), U0, 1.0, max_steps=7)
    assert no == 7
    assert relerr(U7, Uo) <= 1e-10
    Uz, tz, nz = device_run(U0, 0.0, dx=dx)
    assert nz == 0 and tz == 0.0
    assert np.array_equal(Uz, U0)


def test_device_cfl_continues_with_fixed_steps():
    """After rpl_advance_to the current buffer is the last one written."""
    n = (96, 64)
    dx = [1.0 / 96] * 2
    U0 = W.shock_bubble(n, dx=dx)
    with R.Domain(n, dx=dx) as dom:
        dom.set_state(U0)
        t, steps = dom.advance_to(0.01)
        U1 = dom.get_state()
        dom.advance(1e-4, 3)
        U2 = dom.get_state()
    g = oracle.Grid(n, dx=dx)
    Uo, no = oracle.run_cfl(g, U0, 0.01)
    assert steps == no
    assert relerr(U1, Uo) <= 1e-10
    assert relerr(U2, oracle.step(g, U1, 1e-4, 3)) <= 1e-12


def test_device_cfl_domain_error():
    n = (64, 64)
    U0 = W.uniform(n)
    U0[10:20, 10:20, 3] = 0.01   # E below the kinetic energy -> p < 0
    U0[10:20, 10:20, 1] = 1.0
    with R.Domain(n) as dom:
        dom.set_state(U0)
        with pytest.raises(R.DomainError):
            dom.advance_to(0.1)


def _physical(U, gamma=1.4):
    D = U.shape[-1] - 2
    rho = U[..., 0].astype(np.float64)
    ke = 0.5 * np.sum(U[..., 1:1 + D].astype(np.float64) ** 2, axis=-1) / rho
    p = (gamma - 1) * (U[..., D + 1] - ke)
    return bool(np.all(np.isfinite(U)) and rho.min() > 0 and p.min() > 0)


@pytest.mark.parametrize("kernel", ["fused", "split"])
def test_shock_bubble_1000_steps_robust(kernel):
    """SURVEY P9 on the GPU: shock-bubble 512^2 (reading S22), 1000
    device-CFL steps while the shock crosses the bubble -- no domain error, rho, p > 0
    and finite everywhere."""
    n = (512, 512)
    dx = [1.0 / 512] * 2
    U0 = W.shock_bubble(n, dx=dx)
    U, t, steps = device_run(U0, 10.0, max_steps=1000, dx=dx, kernel=kernel)
    assert steps == 1000 and 0.0 < t < 10.0
    assert _physical(U)
    assert U[:, 384:, 0].mean() > 2.0  # the shock has crossed the domain's right half


def test_shock_bubble_1000_steps_matches_oracle():
    """The same 1000-step shock-bubble CFL run at 128^2 against the oracle: same step
    count; the state after the shock-bubble interaction within the north_star bar
    1e-10 (observed 6.8e-15 on the B200, profiles/r1/p9_1000_steps.log)."""
    n = (128, 128)
    dx = [1.0 / 128] * 2
    U0 = W.shock_bubble(n, dx=dx)
    Ug, t, steps = device_run(U0, 10.0, max_steps=1000, dx=dx)
    Uo, no = oracle.run_cfl(oracle.Grid(n, dx=dx), U0, 10.0, max_steps=1000)
    assert steps == no == 1000
    err = relerr(Ug, Uo)
    print(f"1000-step shock-bubble GPU vs oracle: {err:.3e}")
    assert err <= 1e-10
