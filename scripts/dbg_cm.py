"""Probe the column-march 2-D kernel vs the split kernel (debug aid)."""
import os
import subprocess
import sys

SNIP = r'''
import os, sys, numpy as np
sys.path.insert(0, os.environ["ROOT"])
import paper_2104_08571_b200 as R, workloads as W
n = tuple(int(v) for v in os.environ["N"].split(","))
rows = int(os.environ["ROWS"])
dx = [1 / n[0]] * 2
U0 = W.shock_bubble(n, dx=dx)
res = []
for kern in ["fused", "split"]:
    with R.Domain(n, dx=dx, kernel=kern, rows_per_chunk=rows) as d:
        d.set_state(U0); d.advance(1e-5, 1); res.append(d.get_state())
a, b = res
bad = np.argwhere(np.any(a != b, axis=-1))
print("EQUAL" if len(bad) == 0 else f"DIFF n={len(bad)} first={bad[:3].tolist()} last={bad[-3:].tolist()}")
'''
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for var in os.environ.get("VARS", "40").split(","):
    for n in ["130,70", "256,256", "1024,1024"]:
        for rows in [0, 8, 16]:
            env = dict(os.environ, ROOT=root, N=n, ROWS=str(rows), RPL_VARIANT=var)
            r = subprocess.run([sys.executable, "-c", SNIP], env=env, capture_output=True,
                               text=True, timeout=120)
            out = (r.stdout.strip().splitlines() or [""])[-1]
            err = (r.stderr.strip().splitlines() or [""])[-1]
            print(f"v{var} n={n:10s} rows={rows:3d} -> {out} {err[:100] if r.returncode else ''}",
                  flush=True)
