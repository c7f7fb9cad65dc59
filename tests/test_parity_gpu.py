"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerance (BASELINE.json north_star): max relative error <= 1e-10 in fp64 and
<= 1e-4 in fp32 after 100 steps, relative error per component as in DESIGN.md
reading S15: max_i |g - o| / max_i |o|.  Partitioned runs, split vs fused
kernels and AoS vs SoA must be bitwise identical.
"""
import numpy as np
import pytest

import oracle
import paper_2104_08571_b200 as R
import workloads as W

pytestmark = pytest.mark.gpu

OK = {"clamp": oracle.BC_TRANSMISSIVE, "periodic": oracle.BC_PERIODIC,
      "reflective": oracle.BC_REFLECTIVE}


def relerr(g, o):
    """DESIGN.md reading S15: max over components of max|g-o| / max|o|, where the
    momentum components share one scale (max over all momentum components), so a
    transverse momentum that is ~0 everywhere is not divided by itself."""
    C = o.shape[-1]
    o64, g64 = o.astype(np.float64), g.astype(np.float64)
    mom = np.max(np.abs(o64[..., 1:C - 1])) if C > 2 else 0.0
    errs = []
    for c in range(C):
        scale = np.max(np.abs(o64[..., c]))
        if 0 < c < C - 1:
            scale = max(scale, mom)
        diff = np.max(np.abs(g64[..., c] - o64[..., c]))
        errs.append(diff / scale if scale > 0 else diff)
    return max(errs)


def bits_equal(a, b):
    """Bit-pattern equality (np.array_equal treats -0.0 == +0.0; this does not)."""
    it = {4: np.uint32, 8: np.uint64}[a.dtype.itemsize]
    return a.dtype == b.dtype and np.array_equal(a.view(it), b.view(it))


def run_gpu(U0, dt, nsteps, dtype="f64", **kw):
    n = tuple(reversed(U0.shape[:-1]))
    with R.Domain(n, dtype=dtype, **kw) as dom:
        dom.set_state(U0)
        dom.advance(dt, nsteps)
        return dom.get_state()


def run_oracle(U0, dt, nsteps, dx, pad=2, bc_lo=None, bc_hi=None):
    n = tuple(reversed(U0.shape[:-1]))
    D = len(n)
    g = oracle.Grid(n, pad=pad, dx=dx, bc_lo=[OK[b] for b in (bc_lo or ["clamp"] * D)],
                    bc_hi=[OK[b] for b in (bc_hi or ["clamp"] * D)])
    return oracle.step(g, U0, dt, nsteps)


def test_sod_cfl_run_matches_oracle():
    N = 200
    U0 = W.sod(N)
    with R.Domain((N,), pad=2) as dom:
        dom.set_state(U0)
        n = dom.advance_cfl(0.2, cfl=0.9, n_reduced=5, reduce=0.2)
        Ug = dom.get_state()
    Uo, no = oracle.run_cfl(oracle.Grid((N,), pad=2), U0, 0.2)
    assert n == no == 100
    assert relerr(Ug, Uo) <= 1e-10


@pytest.mark.parametrize("kernel", ["fused", "split"])
@pytest.mark.parametrize("workload", ["random", "shock_bubble"])
def test_2d_100_steps_fp64(kernel, workload):
    n = (192, 160)
    dx = [1.0 / 192] * 2
    U0 = W.random_state(n) if workload == "random" else W.shock_bubble(n, dx=dx)
    dt = 0.4 * dx[0] / oracle.max_wavespeed(oracle.Grid(n), U0)
    Ug = run_gpu(U0, dt, 100, kernel=kernel, dx=dx)
    Uo = run_oracle(U0, dt, 100, dx)
    assert relerr(Ug, Uo) <= 1e-10


@pytest.mark.parametrize("bc", ["periodic", "reflective"])
def test_2d_boundary_kinds(bc):
    n = (130, 70)   # ragged: 130 = 2 windows of 62 + 6
    dx = [1.0 / 130] * 2
    U0 = W.random_state(n, seed=3)
    dt = 0.4 * dx[0] / oracle.max_wavespeed(oracle.Grid(n), U0)
    Ug = run_gpu(U0, dt, 60, dx=dx, bc_lo=[bc, bc], bc_hi=[bc, bc])
    Uo = run_oracle(U0, dt, 60, dx, bc_lo=[bc, bc], bc_hi=[bc, bc])
    assert relerr(Ug, Uo) <= 1e-10


def test_3d_fp64():
    n = (28, 24, 20)
    dx = [1.0 / 28] * 3
    U0 = W.shock_bubble(n, dx=dx)
    dt = 0.4 * dx[0] / oracle.max_wavespeed(oracle.Grid(n), U0)
    Ug = run_gpu(U0, dt, 100, dx=dx)
    Uo = run_oracle(U0, dt, 100, dx)
    assert relerr(Ug, Uo) <= 1e-10


def test_3d_mixed_bcs():
    n = (16, 12, 10)
    dx = [1.0 / 16] * 3
    bl = ["reflective", "periodic", "clamp"]
    bh = ["clamp", "periodic", "reflective"]
    U0 = W.random_state(n, seed=5)
    dt = 0.4 * dx[0] / oracle.max_wavespeed(oracle.Grid(n), U0)
    Ug = run_gpu(U0, dt, 50, dx=dx, bc_lo=bl, bc_hi=bh)
    Uo = run_oracle(U0, dt, 50, dx, bc_lo=bl, bc_hi=bh)
    assert relerr(Ug, Uo) <= 1e-10


@pytest.mark.parametrize("n", [(128, 96), (24, 20, 16)])
def test_fp32_against_fp32_oracle(n):
    D = len(n)
    dx = [1.0 / n[0]] * D
    U0 = W.shock_bubble(n, dx=dx).astype(np.float32)
    dt = 0.4 * dx[0] / oracle.max_wavespeed(oracle.Grid(n), U0.astype(np.float64))
    Ug = run_gpu(U0, dt, 100, dtype="f32", dx=dx)
    Uo = run_oracle(U0, dt, 100, dx)
    assert Uo.dtype == np.float32
    assert relerr(Ug, Uo) <= 1e-4


@pytest.mark.parametrize("n,parts", [((128, 96), (2, 2)), ((128, 96), (1, 4)),
                                     ((128, 96), (4, 1)), ((24, 16, 16), (2, 2, 2)),
                                     ((24, 16, 16), (1, 1, 4)), ((200,), (4,))])
@pytest.mark.parametrize("bc", ["clamp", "periodic", "reflective"])
def test_partitioned_bitwise_identical(n, parts, bc):
    D = len(n)
    dx = [1.0 / n[0]] * D
    U0 = W.random_state(n, seed=9)
    dt = 0.3 * dx[0] / 3.0
    kw = dict(dx=dx, bc_lo=[bc] * D, bc_hi=[bc] * D)
    one = run_gpu(U0, dt, 20, **kw)
    many = run_gpu(U0, dt, 20, parts=parts, **kw)
    assert np.array_equal(one, many)


def test_split_fused_and_layouts_bitwise():
    n = (140, 66)
    dx = [1.0 / 140] * 2
    U0 = W.shock_bubble(n, dx=dx)
    dt = 0.4 * dx[0] / 5.8
    a = run_gpu(U0, dt, 30, dx=dx, kernel="fused")
    b = run_gpu(U0, dt, 30, dx=dx, kernel="split")
    c = run_gpu(U0, dt, 30, dx=dx, kernel="split", layout="aos")
    d = run_gpu(U0, dt, 30, dx=dx, kernel="fused", rows_per_chunk=5)
    assert np.array_equal(a, b) and np.array_equal(a, c) and np.array_equal(a, d)


@pytest.mark.parametrize("n,parts", [((20, 12), (2, 3)), ((10, 8, 6), (2, 2, 3))])
def test_fill_padding_halo_soundness(n, parts):
    """After fill_padding every ghost equals the single-block value."""
    D = len(n)
    bl = ["reflective", "periodic", "clamp"][:D]
    bh = ["clamp", "periodic", "reflective"][:D]
    U0 = W.random_state(n, seed=21)
    g = oracle.Grid(n, pad=2, bc_lo=[OK[b] for b in bl], bc_hi=[OK[b] for b in bh])
    P = np.zeros(oracle.padded_shape(g))
    P[tuple(slice(2, 2 + n[d]) for d in reversed(range(D)))] = U0
    P = oracle.fill_ghosts(g, P)
    S = [n[d] // parts[d] for d in range(D)]
    with R.Domain(n, parts=parts, bc_lo=bl, bc_hi=bh) as dom:
        dom.set_state(U0)
        dom.fill_padding()
        for p in range(int(np.prod(parts))):
            pc = np.unravel_index(p, tuple(reversed(parts)))[::-1]
            got = np.moveaxis(dom.get_padded(p), 0, -1)
            sl = tuple(slice(pc[d] * S[d], pc[d] * S[d] + S[d] + 4) for d in reversed(range(D)))
            assert np.array_equal(got, P[sl]), p


def test_ghosts_after_advance_are_sound():
    """The fused kernel's ghost images equal a fresh fill of the same state."""
    n = (130, 40)
    U0 = W.random_state(n, seed=2)
    kw = dict(bc_lo=["reflective", "periodic"], bc_hi=["clamp", "periodic"], parts=(2, 2))
    with R.Domain(n, **kw) as dom:
        dom.set_state(U0)
        dom.advance(1e-4, 3)
        after = [dom.get_padded(p) for p in range(4)]
        dom.set_state(dom.get_state())
        dom.fill_padding()
        fresh = [dom.get_padded(p) for p in range(4)]
    for a, b in zip(after, fresh):
        assert np.array_equal(a, b)


def test_max_wavespeed_matches_oracle():
    for n in [(1000,), (96, 80), (20, 18, 16)]:
        U0 = W.shock_bubble(n, dx=[1.0 / n[0]] * len(n)) if len(n) > 1 else W.sod(n[0])
        with R.Domain(n, parts=(2,) + (1,) * (len(n) - 1)) as dom:
            dom.set_state(U0)
            s = dom.max_wavespeed()
        so = oracle.max_wavespeed(oracle.Grid(n), U0)
        assert abs(s - so) <= 1e-14 * so


def test_domain_error_is_reported():
    n = (64, 64)
    U0 = W.uniform(n)
    U0[..., 3] = -1.0
    with R.Domain(n) as dom:
        dom.set_state(U0)
        dom.advance(1e-3, 1)
        with pytest.raises(R.DomainError):
            dom.synchronize()


@pytest.mark.parametrize("dtype,layout", [("f32", "soa"), ("f32", "aos"), ("f64", "soa")])
@pytest.mark.parametrize("where", ["interior", "corner", "last_row"])
def test_domain_error_is_reported_3d(dtype, layout, where):
    """3-D fused kernels (packed fp32 incl.): one cell with negative pressure -- in the
    interior, at a domain corner, or in the last row half of a packed row pair --
    raises at the next synchronising call; a clean state of the same run does not."""
    n = (40, 30, 20)
    U0 = W.uniform(n, rho=1.0, vel=[0.1, 0.0, -0.2], p=1.0).astype(
        np.float32 if dtype == "f32" else np.float64)
    with R.Domain(n, dtype=dtype, layout=layout) as dom:
        dom.set_state(U0)
        dom.advance(1e-3, 2)
        dom.synchronize()  # clean
    z, y, x = {"interior": (10, 13, 21), "corner": (0, 0, 0), "last_row": (7, 29, 39)}[where]
    U0[z, y, x, 4] = -1.0
    with R.Domain(n, dtype=dtype, layout=layout) as dom:
        dom.set_state(U0)
        dom.advance(1e-3, 1)
        with pytest.raises(R.DomainError):
            dom.synchronize()


def test_uniform_state_bitwise_full_size():
    """BASELINE configs[1] size and launch configuration: uniform state is a fixed point."""
    n = (1024, 1024)
    U0 = W.uniform(n, rho=0.9, vel=[0.4, -0.3], p=1.2)
    Ug = run_gpu(U0, 1e-4, 5)
    assert np.array_equal(Ug, U0)


def _patch_oracle(Uin, lo, hi, n, k, dt, dx, bcs, order=1):
    """Oracle on a sub-box [lo,hi) of the full input; the valid region shrinks by
    (stencil radius) x k per cut side (radius 1 for order 1, 2 for order 2)."""
    D = len(n)
    sl = tuple(slice(lo[d], hi[d]) for d in reversed(range(D)))
    sub = np.ascontiguousarray(Uin[sl])
    pn = tuple(hi[d] - lo[d] for d in range(D))
    g = oracle.Grid(pn, pad=2, dx=dx, bc_lo=[OK[bcs] if lo[d] == 0 else oracle.BC_TRANSMISSIVE
                                             for d in range(D)],
                    bc_hi=[OK[bcs] if hi[d] == n[d] else oracle.BC_TRANSMISSIVE for d in range(D)],
                    order=order)
    out = oracle.step(g, sub, dt, k)
    m = k * order
    v0 = [0 if lo[d] == 0 else m for d in range(D)]
    v1 = [pn[d] if hi[d] == n[d] else pn[d] - m for d in range(D)]
    vsl = tuple(slice(v0[d], v1[d]) for d in reversed(range(D)))
    gsl = tuple(slice(lo[d] + v0[d], lo[d] + v1[d]) for d in reversed(range(D)))
    return out[vsl], gsl


def test_full_size_sampled_parity_2d1024():
    """configs[1] (1024^2 fp64, bench launch config): sampled patches vs the oracle."""
    n = (1024, 1024)
    dx = [1.0 / 1024] * 2
    U0 = W.shock_bubble(n, dx=dx)
    dt = 0.4 * dx[0] / oracle.max_wavespeed(oracle.Grid(n), U0)
    k = 4
    Ug = run_gpu(U0, dt, k, dx=dx)
    for lo in [(0, 0), (980, 0), (90, 500), (400, 440), (1000, 1000), (0, 990), (600, 100)]:
        hi = (min(lo[0] + 44, 1024), min(lo[1] + 44, 1024))
        ref, gsl = _patch_oracle(U0, lo, hi, n, k, dt, dx, "clamp")
        assert relerr(Ug[gsl], ref) <= 1e-12, lo


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("n,rows", [((70, 33, 20), 0), ((70, 33, 20), 5), ((130, 15, 9), 3)])
def test_fused3d_equals_split_bitwise(dtype, n, rows):
    """K-B (3-D, TMA-staged) == K-A (one launch per sweep), ragged tiles, z-chunks."""
    dx = [1.0 / n[0]] * 3
    U0 = W.shock_bubble(n, dx=dx)
    if dtype == "f32":
        U0 = U0.astype(np.float32)
    dt = 0.4 * dx[0] / 5.8
    kw = dict(dx=dx, dtype=dtype, bc_lo=["reflective", "periodic", "clamp"],
              bc_hi=["clamp", "periodic", "reflective"])
    a = run_gpu(U0, dt, 12, kernel="fused", rows_per_chunk=rows, **kw)
    b = run_gpu(U0, dt, 12, kernel="split", **kw)
    assert bits_equal(a, b)


def test_fused3d_partitioned_ghosts_sound():
    n = (40, 30, 24)
    U0 = W.random_state(n, seed=4)
    kw = dict(bc_lo=["reflective", "periodic", "clamp"], bc_hi=["clamp", "periodic", "reflective"],
              parts=(2, 1, 2))
    with R.Domain(n, **kw) as dom:
        dom.set_state(U0)
        dom.advance(1e-4, 3)
        after = [dom.get_padded(p) for p in range(4)]
        dom.set_state(dom.get_state())
        dom.fill_padding()
        fresh = [dom.get_padded(p) for p in range(4)]
    for x, y in zip(after, fresh):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_fused3d_aos_equals_soa_bitwise(dtype):
    """Layout invariance: the AoS ("contiguous") and SoA ("strided")
    storage of the conserved-state struct give bitwise identical steps."""
    n = (66, 30, 18)
    dx = [1.0 / n[0]] * 3
    U0 = W.shock_bubble(n, dx=dx)
    if dtype == "f32":
        U0 = U0.astype(np.float32)
    kw = dict(dx=dx, dtype=dtype, bc_lo=["reflective", "periodic", "clamp"],
              bc_hi=["clamp", "periodic", "reflective"])
    a = run_gpu(U0, 1e-4, 8, layout="soa", **kw)
    b = run_gpu(U0, 1e-4, 8, layout="aos", **kw)
    c = run_gpu(U0, 1e-4, 8, layout="aos", kernel="split", **kw)
    assert np.array_equal(a, b) and np.array_equal(a, c)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("n,pad,parts", [((130, 70), 2, (1, 1)), ((1000, 333), 1, (1, 1)),
                                         ((256, 96), 1, (2, 2))])
def test_flux_difference_tiled_equals_plain_bitwise(dtype, n, pad, parts):
    """f2: the tiled 2-D kernel (each face once) and the paper's per-cell form
    (kernel=split) give bitwise the same R (same operations per face and sum)."""
    dx = [1.0 / n[0]] * 2
    U0 = W.shock_bubble(n, dx=dx)
    if dtype == "f32":
        U0 = U0.astype(np.float32)
    out = []
    for kernel in ("fused", "split"):
        with R.Domain(n, pad=pad, parts=parts, dtype=dtype, dx=dx, kernel=kernel) as dom:
            dom.set_state(U0)
            dom.flux_difference(2e-4)
            out.append(dom.get_flux_difference())
    assert bits_equal(out[0], out[1])


@pytest.mark.parametrize("variant", ["0"])
@pytest.mark.parametrize("parts", [(1, 1), (2, 3)])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_2d_fused_bitwise(parts, dtype, variant, monkeypatch):
    """The 2-D fused kernel gives bitwise the split kernel's result (ragged windows and
    tiles, partitions)."""
    n = (190, 126)
    dx = [1.0 / 190] * 2
    U0 = W.shock_bubble(n, dx=dx)
    if dtype == "f32":
        U0 = U0.astype(np.float32)
    dt = 0.4 * dx[0] / 5.8
    ref = run_gpu(U0, dt, 7, dtype=dtype, kernel="split", dx=dx, parts=parts)
    monkeypatch.setenv("RPL_VARIANT", variant)
    assert bits_equal(run_gpu(U0, dt, 7, dtype=dtype, dx=dx, parts=parts), ref)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_flux_difference_tiled_bitwise_1000x333(dtype):
    """f2 tiled kernel (adjacent row pairs: fp32 packed FFMA2, fp64 double pairs) ==
    per-cell kernel, pad 1, ragged windows and tiles."""
    n = (1000, 333)
    dx = [1.0 / n[0]] * 2
    U0 = W.shock_bubble(n, dx=dx)
    if dtype == "f32":
        U0 = U0.astype(np.float32)
    out = []
    for kernel in ("split", "fused"):
        with R.Domain(n, pad=1, dtype=dtype, dx=dx, kernel=kernel) as dom:
            dom.set_state(U0)
            dom.flux_difference(2e-4)
            out.append(dom.get_flux_difference())
    assert bits_equal(out[0], out[1])


def _sample_boxes(n, size, count, seed):
    """Patch origins: the corners plus seeded interior positions."""
    rng = np.random.default_rng(seed)
    D = len(n)
    out = [tuple(0 for _ in range(D)), tuple(n[d] - size for d in range(D))]
    for _ in range(count):
        out.append(tuple(int(rng.integers(0, n[d] - size + 1)) for d in range(D)))
    return out


@pytest.mark.parametrize("n,dtype,tol", [((512, 512, 512), "f64", 1e-12),
                                         ((384, 384, 384), "f32", 1e-4)])
def test_full_size_sampled_parity_3d(n, dtype, tol):
    """BASELINE configs[2] (512^3 fp64) and configs[3] (384^3 fp32 per GPU) at full size in
    the bench's launch configuration: 2 fused steps, sampled 20^3 patches vs the oracle."""
    dx = [1.0 / n[0]] * 3
    U0 = W.shock_bubble(n, dx=dx)
    if dtype == "f32":
        U0 = U0.astype(np.float32)
    dt = 0.4 * dx[0] / 5.8
    k = 2
    Ug = run_gpu(U0, dt, k, dtype=dtype, dx=dx)
    for lo in _sample_boxes(n, 20, 4, seed=7) + [(40, n[1] // 2 - 10, n[2] // 2 - 10)]:
        hi = tuple(lo[d] + 20 for d in range(3))
        ref, gsl = _patch_oracle(U0, lo, hi, n, k, dt, dx, "clamp")
        assert relerr(Ug[gsl], ref) <= tol, lo


def test_full_size_sampled_parity_order2_2d1024():
    """f3 at configs[1] size: order-2 fused kernel, sampled patches vs the order-2 oracle."""
    n = (1024, 1024)
    dx = [1.0 / 1024] * 2
    U0 = W.shock_bubble(n, dx=dx)
    dt = 0.4 * dx[0] / 5.8
    k = 3
    with R.Domain(n, dx=dx, order=2) as dom:
        dom.set_state(U0)
        dom.advance(dt, k)
        Ug = dom.get_state()
    for lo in _sample_boxes(n, 48, 5, seed=3) + [(80, 480)]:
        hi = (lo[0] + 48, lo[1] + 48)
        ref, gsl = _patch_oracle(U0, lo, hi, n, k, dt, dx, "clamp", order=2)
        assert relerr(Ug[gsl], ref) <= 1e-12, lo


@pytest.mark.parametrize("variant,dtype", [("0", "f32"), ("1", "f32"), ("0", "f64"), ("1", "f64")])
def test_3d_kernel_variants_bitwise(variant, dtype, monkeypatch):
    """3-D fused kernels (RPL_VARIANT 0 = default: fp64 k_step3d_sp, fp32 k_step3d_rb;
    1 = the other form) give bitwise the split kernel's result (ragged windows, tiles
    and z-chunks)."""
    n = (70, 33, 20)
    dx = [1.0 / 70] * 3
    U0 = W.shock_bubble(n, dx=dx)
    if dtype == "f32":
        U0 = U0.astype(np.float32)
    dt = 0.4 * dx[0] / 5.8
    ref = run_gpu(U0, dt, 5, dtype=dtype, kernel="split", dx=dx, rows_per_chunk=7)
    monkeypatch.setenv("RPL_VARIANT", variant)
    assert bits_equal(run_gpu(U0, dt, 5, dtype=dtype, dx=dx, rows_per_chunk=7), ref)


def test_configs1_full_field_100_steps():
    """BASELINE configs[1] exactly as north_star states the bar: 2-D 1024^2 fp64, 100
    steps on the GPU (bench launch configuration) vs the oracle over the whole field,
    max relative error <= 1e-10 (reading S15 metric)."""
    n = (1024, 1024)
    dx = [1.0 / 1024] * 2
    U0 = W.shock_bubble(n, dx=dx)
    dt = 0.4 * dx[0] / oracle.max_wavespeed(oracle.Grid(n), U0)
    Ug = run_gpu(U0, dt, 100, dx=dx)
    Uo = run_oracle(U0, dt, 100, dx)
    assert relerr(Ug, Uo) <= 1e-10


@pytest.mark.parametrize("n", [(2,), (3,), (2, 2), (3, 2), (2, 5, 3), (2, 2, 2)])
@pytest.mark.parametrize("bc", ["clamp", "periodic", "reflective"])
@pytest.mark.parametrize("kernel", ["fused", "split"])
def test_minimum_sizes(n, bc, kernel):
    """Degenerate extents: every dim exactly pad (2) or just above -- the windows,
    tiles and z-chunks are almost all halo, every cell is a boundary cell."""
    D = len(n)
    dx = [1.0 / 8] * D
    U0 = W.random_state(n, seed=17)
    dt = 0.2 * dx[0] / 3.0
    kw = dict(bc_lo=[bc] * D, bc_hi=[bc] * D)
    Ug = run_gpu(U0, dt, 4, dx=dx, kernel=kernel, **kw)
    Uo = run_oracle(U0, dt, 4, dx, **kw)
    assert relerr(Ug, Uo) <= 1e-10


@pytest.mark.parametrize("n", [(2, 2, 2), (3, 2, 5), (2, 17, 3), (31, 15, 2), (33, 16, 17)])
@pytest.mark.parametrize("bc", ["clamp", "periodic", "reflective"])
@pytest.mark.parametrize("layout", ["soa", "aos"])
def test_minimum_sizes_fp32_packed(n, bc, layout):
    """The packed fp32 3-D kernel (two tile rows per lane) at degenerate and
    tile-edge extents (one row pair half empty, x just past one window, y just
    past one 14-row tile): bit pattern of the split kernel, and the fp32 oracle."""
    D = 3
    dx = [1.0 / 8] * D
    U0 = W.random_state(n, seed=19).astype(np.float32)
    dt = 0.2 * dx[0] / 3.0
    kw = dict(bc_lo=[bc] * D, bc_hi=[bc] * D)
    Ug = run_gpu(U0, dt, 4, dtype="f32", dx=dx, layout=layout, **kw)
    Us = run_gpu(U0, dt, 4, dtype="f32", dx=dx, kernel="split", **kw)
    assert bits_equal(Ug, Us)
    Uo = run_oracle(U0, dt, 4, dx, **kw)
    assert relerr(Ug, Uo) <= 1e-4


def test_zero_steps_and_repeated_calls_compose():
    """advance(dt, 0) is a no-op; advance(dt, 3) == three advance(dt, 1) calls (bitwise)."""
    n = (70, 40)
    dx = [1.0 / 70] * 2
    U0 = W.shock_bubble(n, dx=dx)
    dt = 0.4 * dx[0] / 5.8
    with R.Domain(n, dx=dx) as dom:
        dom.set_state(U0)
        dom.advance(dt, 0)
        assert np.array_equal(dom.get_state(), U0)
        dom.advance(dt, 3)
        a = dom.get_state()
    with R.Domain(n, dx=dx) as dom:
        dom.set_state(U0)
        for _ in range(3):
            dom.advance(dt, 1)
        b = dom.get_state()
    assert np.array_equal(a, b)


@pytest.mark.parametrize("n,parts", [((190, 126), (2, 3)), ((40, 34, 24), (1, 2, 2))])
def test_fault_hook_turns_partition_bitwise_red(n, parts, monkeypatch):
    """RPL_FAULT_HALO=1 (tests only) flips one mantissa bit (2^-20 relative) of rho in one halo
    ghost of every partition after each step: the multi-partition vs one-partition bit
    identity must break (the bitwise tests can fail), while a one-partition run (no halo
    exchange) is untouched."""
    D = len(n)
    dx = [1.0 / n[0]] * D
    U0 = W.shock_bubble(n, dx=dx)
    dt = 0.4 * dx[0] / 5.8
    ref = run_gpu(U0, dt, 5, dx=dx)
    assert np.array_equal(run_gpu(U0, dt, 5, dx=dx, parts=parts), ref)
    monkeypatch.setenv("RPL_FAULT_HALO", "1")
    assert not np.array_equal(run_gpu(U0, dt, 5, dx=dx, parts=parts), ref)
    assert np.array_equal(run_gpu(U0, dt, 5, dx=dx), ref)
