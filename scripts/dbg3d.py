"""Probe the 3-D fused kernel across sizes / variants in subprocesses (debug aid)."""
import itertools
import os
import subprocess
import sys

SNIP = r'''
import os, sys, numpy as np
sys.path.insert(0, os.environ["ROOT"])
import paper_2104_08571_b200 as R, workloads as W
n = tuple(int(v) for v in os.environ["N"].split(","))
dt = os.environ["DT"]; rows = int(os.environ["ROWS"])
dx = [1 / n[0]] * 3
U0 = W.shock_bubble(n, dx=dx).astype(np.float32 if dt == "f32" else np.float64)
with R.Domain(n, dtype=dt, dx=dx, kernel="fused", rows_per_chunk=rows) as d:
    d.set_state(U0); d.advance(1e-4, 2); a = d.get_state()
with R.Domain(n, dtype=dt, dx=dx, kernel="split") as d:
    d.set_state(U0); d.advance(1e-4, 2); b = d.get_state()
print("EQUAL" if np.array_equal(a, b) else "DIFF %g" % np.max(np.abs(a - b)))
'''
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for (n, dt, rows, var) in itertools.product(["24,20,16", "70,33,20", "70,20,16", "24,33,16", "130,20,10"],
                                            ["f32", "f64"], [0, 4], ["", "20"]):
    if dt == "f64" and var:
        continue
    env = dict(os.environ, ROOT=root, N=n, DT=dt, ROWS=str(rows), RPL_VARIANT=var,
               CUDA_LAUNCH_BLOCKING="1")
    r = subprocess.run([sys.executable, "-c", SNIP], env=env, capture_output=True, text=True,
                       timeout=120)
    out = (r.stdout.strip().splitlines() or [""])[-1]
    err = (r.stderr.strip().splitlines() or [""])[-1]
    print(f"n={n:10s} {dt} rows={rows} var={var or '-':2s} -> {out} {err[:120] if r.returncode else ''}",
          flush=True)
