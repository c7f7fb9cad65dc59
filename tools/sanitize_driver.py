"""Small runs of every step kernel for compute-sanitizer (racecheck / synccheck /
memcheck): python tools/sanitize_driver.py CASE, CASE in
  2d       k_step2d_ra<pd> (fp64) and <pk> (fp32), 2 partitions (images into a peer)
  3d64     k_step3d_sp<pd> (default fp64) + k_step3d_rb<pd> (variant 1)
  3d32     k_step3d_rb<pk> (default fp32) + k_step3d_sp<pk> (variant 1), SoA and AoS
  o2       order 2: k_step2d_o2 (2-D), k_step2d_o2<3> + k_zmarch2 (3-D)
  fd       flux difference: k_fluxdiff_ra<pd>/<pk> (tiled) and k_fluxdiff (per cell)
  cfl      device CFL (wavespeed epilogue + step_coef) in 2-D and 3-D
  split    k_sweep / k_sweep2 / k_fill / k_maxws
Grids span several tiles, windows and z-chunks with ragged edges."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_08571_b200 as R  # noqa: E402
import workloads as W  # noqa: E402


def run(n, steps=2, dtype="f64", env=None, **kw):
    old = dict(os.environ)
    os.environ.update(env or {})
    try:
        D = len(n)
        dx = [1.0 / n[0]] * D
        U = W.shock_bubble(n, dx=dx)
        if dtype == "f32":
            U = U.astype(np.float32)
        with R.Domain(n, dx=dx, dtype=dtype, **kw) as dom:
            dom.set_state(U)
            s = dom.max_wavespeed()
            dom.advance(0.4 * dx[0] / s, steps)
            dom.synchronize()
            return dom.get_state()
    finally:
        os.environ.clear()
        os.environ.update(old)


def main(case):
    if case == "2d":
        run((70, 40), parts=(1, 2))
        run((70, 40), dtype="f32")
    elif case == "3d64":
        run((40, 20, 20), rows_per_chunk=8)
        run((40, 20, 20), rows_per_chunk=8, env={"RPL_VARIANT": "1"})
    elif case == "3d32":
        run((40, 20, 20), dtype="f32", rows_per_chunk=8)
        run((40, 20, 20), dtype="f32", rows_per_chunk=8, layout="aos")
        run((40, 20, 20), dtype="f32", rows_per_chunk=8, env={"RPL_VARIANT": "1"})
    elif case == "o2":
        run((70, 40), order=2)
        run((40, 20, 12), order=2)
    elif case == "fd":
        for dtype in ("f64", "f32"):
            n = (70, 40)
            dx = [1.0 / 70] * 2
            U = W.shock_bubble(n, dx=dx)
            if dtype == "f32":
                U = U.astype(np.float32)
            for kernel in ("fused", "split"):
                with R.Domain(n, pad=1, dtype=dtype, dx=dx, kernel=kernel) as dom:
                    dom.set_state(U)
                    dom.flux_difference(1e-4)
                    dom.get_flux_difference()
    elif case == "cfl":
        for n in ((70, 40), (40, 20, 20)):
            dx = [1.0 / n[0]] * len(n)
            with R.Domain(n, dx=dx) as dom:
                dom.set_state(W.shock_bubble(n, dx=dx))
                dom.advance_to(1.0, max_steps=3)
    elif case == "split":
        run((70, 40), kernel="split")
        run((40, 20, 12), kernel="split", order=2)
    else:
        raise SystemExit(f"unknown case {case}")
    print(f"{case} ok")


if __name__ == "__main__":
    main(sys.argv[1])
