"""Per-launch time of the 2-D step kernel across grid sizes (L2 flushed between
launches, rpl_profile CUDA events): where the fixed per-launch cost of small grids
shows.  usage: python scripts/size_sweep.py [sizes...]   (e.g. 1024 2048 4096)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2104_08571_b200 as R
import workloads as W

sizes = [int(a) for a in sys.argv[1:]] or [512, 1024, 1536, 2048, 3072, 4096, 6400]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(64 << 20, dtype=torch.float32, device="cuda")  # 256 MiB read
acc = torch.zeros((), dtype=torch.float32, device="cuda")


def do_flush():
    # bench.py's flush: write 256 MiB, then read 256 MiB so the L2 holds clean lines
    flush.fill_(1)
    acc.add_(flush_rd.sum())

peak = 6542.7
for n in sizes:
    shape = (n, n)
    dx = [1.0 / n] * 2
    with R.Domain(shape, pad=2, dtype="f64", dx=dx, device=0,
                  stream=torch.cuda.current_stream().cuda_stream) as dom:
        dom.set_state(W.shock_bubble(shape, dx=dx))
        dt = 0.4 * dx[0] / dom.max_wavespeed()
        for _ in range(3):
            do_flush()
            dom.advance(dt, 1)
        dom.profile(1000)
        dom.profile_read()
        k = 20
        torch.cuda.synchronize()
        torch.cuda._sleep(200_000 * k)  # GPU head start: events time the device, not launch latency
        for _ in range(k):
            do_flush()
            dom.advance(dt, 1)
        ms, cnt = dom.profile_read()
        t = ms / cnt * 1e3
        cells = n * n
        frac = 64.0 * cells / (t * 1e-6) / 1e9 / peak
        print(f"{n}x{n}: {t:8.2f} us/launch  {t * 1e6 / cells:6.2f} ps/cell  "
              f"HBM frac {frac:.3f}  ({os.environ.get('RPL_VARIANT', '0')})", flush=True)
