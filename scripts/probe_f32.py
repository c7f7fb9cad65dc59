"""Probe fp32 code paths one by one in subprocesses (debug aid)."""
import os
import subprocess
import sys

SNIP = r'''
import os, sys, numpy as np
sys.path.insert(0, os.environ["ROOT"])
import paper_2104_08571_b200 as R, workloads as W
case = os.environ["CASE"]; dt = os.environ["DT"]
n = {"3": (24, 20, 16), "2": (70, 40), "1": (100,)}[case[0]]
D = len(n); dx = [1 / n[0]] * D
U0 = (W.shock_bubble(n, dx=dx) if D > 1 else W.sod(n[0])).astype(np.float32 if dt == "f32" else np.float64)
kern = "split" if "split" in case else "fused"
with R.Domain(n, dtype=dt, dx=dx, kernel=kern) as d:
    d.set_state(U0)
    if "get" in case: d.get_state()
    if "fill" in case: d.fill_padding(); d.synchronize()
    if "mws" in case: d.max_wavespeed()
    if "adv" in case: d.advance(1e-4, 1); d.synchronize()
print("OK")
'''
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for dt in ["f32", "f64"]:
    for case in ["3get", "3fill", "3mws", "3adv_split", "3adv_fused", "2adv_split", "2adv_fused",
                 "1adv_split"]:
        env = dict(os.environ, ROOT=root, CASE=case, DT=dt, CUDA_LAUNCH_BLOCKING="1")
        r = subprocess.run([sys.executable, "-c", SNIP], env=env, capture_output=True, text=True,
                           timeout=120)
        out = (r.stdout.strip().splitlines() or [""])[-1]
        err = (r.stderr.strip().splitlines() or [""])[-1]
        print(f"{dt} {case:12s} -> {out} {err[:150] if r.returncode else ''}", flush=True)
