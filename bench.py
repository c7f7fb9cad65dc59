#!/usr/bin/env python
"""bench.py -- throughput of the split FORCE step (Ripple, arXiv 2104.08571) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--workload 2d1024|s512|w384|l256] [--kernel fused|split]

Metric (BASELINE.json): Gcell-updates/s = global interior cells x steps / time / 1e9,
plus the HBM-roofline fraction of the dominant kernel.

Default workload = BASELINE.json configs[1]: 2-D Euler, 1024 x 1024 cells per GPU,
pad 2, fp64, SoA, shock-bubble initial data (workloads.shock_bubble), fixed
dt = 0.4 dx / S0.  At N > 1 (torchrun, one process per GPU, NCCL) the grid grows
in y (1024 x 1024N, y-split into N partitions: the paper's weak-scaling setup,
P:1393-1402) -> "scaling": "weak".  The two 33.5 MB state buffers fit in the
126 MB L2, so L2 is flushed (256 MiB write) between timed steps and each step is
timed with its own CUDA events on the library's stream (flush excluded).

Only the --impl reference leg and the cpu_baseline object execute oracle/ (the
plain-C CPU oracle, timed as a reported baseline, never the product path).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: ndim, per-GPU (weak) or global (strong) size, dtype, scaling, config label
    "2d1024": dict(ndim=2, n=(1024, 1024), dtype="f64", scaling="weak",
                   label="2-D Euler FORCE 1024x1024/GPU pad 2 fp64 (BASELINE configs[1])"),
    "s512": dict(ndim=3, n=(512, 512, 512), dtype="f64", scaling="strong",
                 label="3-D Euler FORCE 512^3 fp64 z-slabs (BASELINE configs[2])"),
    "w384": dict(ndim=3, n=(384, 384, 384), dtype="f32", scaling="weak",
                 label="3-D Euler FORCE 384^3/GPU fp32 blocks (BASELINE configs[3])"),
    "l256": dict(ndim=3, n=(256, 256, 256), dtype="f32", scaling="weak",
                 label="3-D Euler FORCE 256^3 (BASELINE configs[4])"),
    # the paper's own 2-D scaling problems
    "p6400": dict(ndim=2, n=(6400, 4000), dtype="f64", scaling="strong",
                  label="2-D Euler FORCE 6400x4000 fp64, y-split (paper strong 'small', P:1407)"),
    "p9600": dict(ndim=2, n=(9600, 6000), dtype="f64", scaling="strong",
                  label="2-D Euler FORCE 9600x6000 fp64, y-split (paper strong 'large', P:1408)"),
    "pweak": dict(ndim=2, n=(2560, 2500), dtype="f64", scaling="weak",
                  label="2-D Euler FORCE 6.4M cells/GPU fp64, y-split (paper weak, P:1393-1402)"),
    # order-2 reconstruction (MUSCL-Hancock + FORCE), configs[1] shape
    "o2_1024": dict(ndim=2, n=(1024, 1024), dtype="f64", scaling="weak", order=2,
                    label="2-D Euler SLIC (MUSCL-Hancock + FORCE, order 2) 1024x1024/GPU fp64"),
    "o2_s256": dict(ndim=3, n=(256, 256, 256), dtype="f64", scaling="weak", order=2,
                    label="3-D Euler SLIC (order 2) 256^3 fp64 (x-y pass + z pass)"),
    # CFL-adaptive steps (Listing 8 wavespeed -> max -> dt every step);
    # one bench "step" = one run of cfl_steps CFL steps (--cfl-loop device|host)
    "cfl1024": dict(ndim=2, n=(1024, 1024), dtype="f64", scaling="weak", op="cfl", cfl_steps=20,
                    label="2-D Euler FORCE 1024x1024/GPU fp64, CFL-adaptive dt (20 steps/run)"),
    "cfl6400": dict(ndim=2, n=(6400, 4000), dtype="f64", scaling="strong", op="cfl",
                    cfl_steps=10,
                    label="2-D Euler FORCE 6400x4000 fp64, CFL-adaptive dt (10 steps/run)"),
}
# the paper's Table 4 (sec. 7.3) flux difference, strided layout,
# one pass over (k*1024)^2 cells; paper V100 times (ms) as context.
PAPER_TABLE4_MS = {1: 0.0757, 2: 0.2438, 4: 0.9101, 8: 3.5533, 16: 14.282, 32: 59.028}
for _k in PAPER_TABLE4_MS:
    WORKLOADS[f"fd{_k}k"] = dict(
        ndim=2, n=(_k * 1024, _k * 1024), dtype="f32", scaling="weak", op="fluxdiff",
        pad=1, paper_ms=PAPER_TABLE4_MS[_k],
        label=f"sec. 7.3 flux difference {_k}k^2 fp32 SoA (paper Table 4, Size^2 = {_k}k)")
W384_BLOCKS = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}


def decomposition(wl, nranks):
    """Global size and partition grid for N ranks."""
    n = list(wl["n"])
    D = wl["ndim"]
    if wl["scaling"] == "strong":
        parts = [1] * D
        parts[D - 1] = nranks
        return n, parts
    if D == 3 and nranks in W384_BLOCKS:
        parts = list(W384_BLOCKS[nranks])
    else:
        parts = [1] * D
        parts[D - 1] = nranks
    return [n[d] * parts[d] for d in range(D)], parts


class Clocks:
    """Sample SM clocks and clock-event (throttle) reasons during the timed region:
    NVML polled every ~2 ms (the timed region of a short run lasts milliseconds),
    nvidia-smi every 100 ms as the fallback."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clock-event reason bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40}

    def __init__(self, index):
        self.index = index
        self.samples = []   # (sm_mhz, max_mhz, set(reasons))
        self.source = None
        self._stop = threading.Event()
        self._t = None
        self._nv = None

    def _nvml_handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        props = torch.cuda.get_device_properties(self.index)
        for i in range(pynvml.nvmlDeviceGetCount()):
            h = pynvml.nvmlDeviceGetHandleByIndex(i)
            pci = pynvml.nvmlDeviceGetPciInfo(h)
            if pci.bus == props.pci_bus_id and pci.device == props.pci_device_id:
                return pynvml, h
        return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _run(self):
        try:
            nv, h = self._nvml_handle()
            get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.source = "nvml"
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = get_r(h)
                self.samples.append((float(sm), float(mx),
                                     {k for k, bit in self.BITS.items() if r & bit}))
                self._stop.wait(0.002)
            return
        except Exception:
            self.samples = []
        self.source = "nvidia-smi"
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout
                f = [v.strip() for v in out.strip().split(",")]
                if len(f) >= 7 and f[0].replace(".", "").isdigit():
                    self.samples.append((float(f[0]), float(f[1]),
                                         {names[i] for i in range(4)
                                          if f[3 + i].lower() == "active"}))
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.05)  # first samples before the timed region starts
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted(set().union(*[s[2] for s in self.samples]))
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples), "source": self.source}


def N_get_fd(dom, ptr):
    """rpl_get_flux_difference into a raw host pointer (e2e of the flux-difference op)."""
    import ctypes

    from paper_2104_08571_b200 import _native as N
    N.check(N.lib().rpl_get_flux_difference(dom._h, ctypes.c_void_p(ptr)))


def measured_peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(key):
    """dram bytes read+write per launch of the dominant kernel, from the committed
    ncu --set full capture summary (profiles/ncu_traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def cpu_baseline(wl, steps_cap=60, budget_s=12.0):
    """The oracle as it stands (plain C, 1 thread) on a bounded sample of the workload."""
    import numpy as np  # noqa

    import oracle
    import workloads as W
    D = wl["ndim"]
    n = list(wl["n"])
    if D == 3:  # bounded sample: a 128^3 sub-box of the same recipe
        n = [128, 128, 128]
    elif n[0] * n[1] > 2048 * 2048:  # bounded sample: a 2048^2 sub-box
        n = [2048, 2048]
    dx = [1.0 / wl["n"][0]] * D
    U = W.shock_bubble(tuple(n), dx=dx)
    if wl["dtype"] == "f32":
        U = U.astype(np.float32)
    op = wl.get("op", "step")
    g = oracle.Grid(tuple(n), pad=wl.get("pad", 2), dx=dx, order=wl.get("order", 1))
    dt = 0.4 * dx[0] / oracle.max_wavespeed(g, U.astype(np.float64))

    def run(k):
        if op == "fluxdiff":  # one flux-difference pass per "step" (Table 4 kernel)
            for _ in range(k):
                oracle.flux_difference(g, U, dt)
        elif op == "cfl":  # the oracle's CFL loop (wavespeed pass + dt every step)
            oracle.run_cfl(g, U, 1e9, cfl=0.9, n_reduced=0, max_steps=k)
        else:
            oracle.step(g, U, dt, k)

    t0 = time.perf_counter()
    run(1)
    one = time.perf_counter() - t0
    k = max(1, min(steps_cap, int(budget_s / max(one, 1e-6))))
    t0 = time.perf_counter()
    run(k)
    el = time.perf_counter() - t0
    cells = int(np.prod(n))
    unit = "Gcell/s" if op == "fluxdiff" else "Gcell-updates/s"
    what = {"fluxdiff": "flux-difference passes", "cfl": "CFL steps"}.get(op, "steps")
    return {"value": cells * k / el / 1e9, "unit": unit, "cores": 1,
            "kind": "oracle",
            "sample": f"{'x'.join(map(str, n))} shock-bubble {wl['dtype']}"
                      f"{' order 2' if wl.get('order', 1) == 2 else ''}, {k} {what}, "
                      f"plain-C oracle single thread ({el:.1f} s)"}


def run_reference(args, wl):
    """--impl reference: the oracle on this arm's config/metric (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    import workloads as W
    D = wl["ndim"]
    n = list(wl["n"])
    full = int(np.prod(n))
    sample_n = n if full <= 2 ** 20 else [min(v, 128) for v in n]
    dx = [1.0 / n[0]] * D
    U = W.shock_bubble(tuple(sample_n), dx=dx)
    if wl["dtype"] == "f32":
        U = U.astype(np.float32)
    g = oracle.Grid(tuple(sample_n), pad=2, dx=dx, order=wl.get("order", 1))
    dt = 0.4 * dx[0] / oracle.max_wavespeed(g, U.astype(np.float64))
    for _ in range(args.warmup):
        U = oracle.step(g, U, dt, 1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        U = oracle.step(g, U, dt, 1)
    el = time.perf_counter() - t0
    cells = int(np.prod(sample_n))
    value = cells * args.steps / el / 1e9
    sample = (f"{'x'.join(map(str, sample_n))} of the workload per step "
              f"({'full grid' if sample_n == n else 'sub-box'}), plain-C oracle, 1 thread")
    line = {"impl": "reference", "metric": "Gcell-updates/s", "value": value,
            "unit": "Gcell-updates/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
            "higher_is_better": True, "scaling": wl["scaling"], "vs_baseline": None,
            "dtype": wl["dtype"], "data": "synthetic",
            "config": {"workload": wl["label"], "sample": sample},
            "cpu_baseline": {"value": value, "unit": "Gcell-updates/s", "cores": 1,
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "Gcell-updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="2d1024", choices=sorted(WORKLOADS))
    ap.add_argument("--cfl-loop", default="device", choices=["device", "host"],
                    help="cfl workloads: rpl_advance_to (device-side dt) or rpl_advance_cfl "
                         "(host loop: wavespeed pass + sync every step)")
    ap.add_argument("--kernel", default="fused", choices=["fused", "split"])
    ap.add_argument("--dtype", default=None, choices=["f32", "f64"],
                    help="override the workload's dtype (configs[4] runs both)")
    ap.add_argument("--layout", default="soa", choices=["soa", "aos"],
                    help="HBM layout of the conserved-state struct (BASELINE configs[4])")
    ap.add_argument("--rows", type=int, default=0, help="rows per warp task (0 = auto)")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="halo transport between ranks (N > 1): P2P = step kernels store halos "
                         "into the neighbour's buffer over NVLink (CUDA IPC); NCCL = pack + "
                         "ncclSend/Recv + unpack")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    wl = dict(WORKLOADS[args.workload])
    if args.dtype:
        wl["dtype"] = args.dtype
    if args.impl == "reference":
        return run_reference(args, wl)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2104_08571_b200 as R
    import workloads as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # RPL_SHARE_DEVICE=1: every rank on cuda:0 (functional check of the N>1 path on
    # a 1-GPU box; timings are then meaningless: the processes time-slice one GPU)
    share = os.environ.get("RPL_SHARE_DEVICE") == "1"
    # torch.distributed over NCCL for the plumbing (ncclUniqueId broadcast, IPC-handle
    # all-gather, max-over-ranks timing); gloo only when all ranks share one GPU
    # (NCCL rejects two ranks on one device)
    backend = "gloo" if share else "nccl"
    if share and args.transport == "nccl":
        raise SystemExit("RPL_SHARE_DEVICE=1 needs --transport p2p (NCCL: one rank per GPU)")
    if world > 1:
        torch.cuda.set_device(0 if share else local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    # a real (non-default) stream shared by the library, the events and the L2 flush
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    gn, parts = decomposition(wl, world)
    D = wl["ndim"]
    dx = [1.0 / wl["n"][0]] * D
    nccl_id = None
    if world > 1 and args.transport == "nccl":
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(R.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().numpy().tobytes())
    op = wl.get("op", "step")
    dom = R.Domain(gn, pad=wl.get("pad", 2), parts=parts, dtype=wl["dtype"], kernel=args.kernel,
                   dx=dx,
                   layout=args.layout,
                   nranks=world, rank=rank if world > 1 else 0, nccl_id=nccl_id, device=dev,
                   stream=stream.cuda_stream, rows_per_chunk=args.rows,
                   transport=args.transport if world > 1 else "nccl", order=wl.get("order", 1))
    if world > 1 and args.transport == "p2p":
        blobs = [None] * world
        dist.all_gather_object(blobs, dom.p2p_export())
        dom.p2p_attach(blobs)
    box = (dom.lo, dom.hi)
    U0 = W.shock_bubble(tuple(gn), dx=dx, box=box)
    if wl["dtype"] == "f32":
        U0 = U0.astype(np.float32)
    dom.set_state(U0)
    S0 = dom.max_wavespeed()
    dt = 0.4 * min(dx) / S0
    local_cells = int(np.prod([dom.box[d] for d in range(D)]))
    global_cells = int(np.prod(gn))
    elem = 8 if wl["dtype"] == "f64" else 4
    C = D + 2

    flush = None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush_rd = None if args.no_flush else torch.ones(32 << 20, dtype=torch.float64, device="cuda")
    flush_acc = torch.zeros((), dtype=torch.float64, device="cuda")

    def do_flush():
        # write 256 MiB (evicts the state from the 126 MB L2), then read another
        # 256 MiB so the L2 holds clean lines: the next step pays no write-backs
        # of the flush buffer
        if flush is not None:
            flush.fill_(1)
            flush_acc.add_(flush_rd.sum())

    for _ in range(args.warmup):
        dom.advance(dt, 1)
        do_flush()
    torch.cuda.synchronize()

    launches_per_step = dom.launches_per_step
    M = wl.get("cfl_steps", 1)

    def run_cfl():
        # t_end far away: every run takes exactly M steps (the max_steps bound)
        if args.cfl_loop == "device":
            t, n = dom.advance_to(1e9, cfl=0.9, n_reduced=0, max_steps=M)
        else:
            n = dom.advance_cfl(1e9, cfl=0.9, n_reduced=0, max_steps=M)
        assert n == M, n

    def timed_loop(nsteps, profile):
        """nsteps steps, each bracketed by CUDA events on the library stream, L2
        flushed between steps (outside the events).  With profile=True the library
        also brackets every step-kernel launch with its own events (rpl_profile)."""
        if profile:
            dom.profile(nsteps * 64)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(nsteps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        # GPU-side head start so the host queues the steps ahead of the GPU:
        # the step events then measure device time, not host launch latency
        if op != "cfl":  # (a CFL run synchronises inside: it includes its host latency)
            torch.cuda._sleep(200_000 * nsteps)
        for k in range(nsteps):
            ev[k][0].record(stream)
            if op == "fluxdiff":
                dom.flux_difference(dt)
            elif op == "cfl":
                run_cfl()
            else:
                dom.advance(dt, 1)
            ev[k][1].record(stream)
            do_flush()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        kern = dom.profile_read() if profile else (0.0, 0)
        if profile:
            dom.profile(0)
        per_step = [a.elapsed_time(b) for a, b in ev]  # ms
        timed_loop.last_steps = per_step
        return sum(per_step) / 1e3, kern

    wall0 = time.perf_counter()
    with Clocks(dev) as clk:
        t_total, _ = timed_loop(args.steps, profile=False)   # the headline timing
    step_list = list(timed_loop.last_steps)
    wall = time.perf_counter() - wall0
    # the dominant kernel's own launch time for the roofline (separate, profiled pass)
    n_prof = max(5, min(args.steps, 20))
    t_prof, (kern_ms, kern_launches) = timed_loop(n_prof, profile=True)
    # exposed halo / synchronisation time per step: the step's event time minus its
    # step-kernel time (pack/unpack, NCCL, P2P flag kernel, launch gaps)
    exposed_ms = max(0.0, (t_prof * 1e3 - kern_ms) / n_prof)
    if world > 1:
        tt = torch.tensor([t_total], dtype=torch.float64,
                          device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total = float(tt.item())
        ts = torch.tensor(step_list, dtype=torch.float64,
                          device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(ts, op=dist.ReduceOp.MAX)
        step_list = ts.cpu().tolist()
    dom.synchronize()  # surfaces any domain error of the timed steps

    # ---- e2e through the public API with host buffers (pinned), copies timed
    e2e = None
    if args.e2e_steps > 0:
        tdt = torch.float64 if elem == 8 else torch.float32
        h_in = torch.empty(C * local_cells, dtype=tdt, pin_memory=True)
        h_out = torch.empty(C * local_cells, dtype=tdt, pin_memory=True)
        h_in.numpy()[:] = np.ascontiguousarray(np.moveaxis(U0, -1, 0)).ravel()
        dom.get_state_ptr(h_out.data_ptr())
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            dom.set_state_ptr(h_in.data_ptr())
            if op == "fluxdiff":
                dom.flux_difference(dt)
                N_get_fd(dom, h_out.data_ptr())
            elif op == "cfl":
                run_cfl()
                dom.get_state_ptr(h_out.data_ptr())
            else:
                dom.advance(dt, 1)
                dom.get_state_ptr(h_out.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize()
        te = e0.elapsed_time(e1) / 1e3
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64,
                              device="cuda" if backend == "nccl" else "cpu")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        nb = C * local_cells * elem
        e2e = {"value": global_cells * M * args.e2e_steps / te / 1e9, "unit": "Gcell-updates/s",
               "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb, "steps": args.e2e_steps,
               "path": "rpl_set_state(pinned host) + rpl_advance(dt,1) + rpl_get_state(pinned host)"}

    value = global_cells * M * args.steps / t_total / 1e9
    if op == "cfl":
        # device loop: M step launches + the initial wavespeed pass; host loop: a
        # wavespeed pass before every step
        launches_per_step = M * launches_per_step + (1 if args.cfl_loop == "device" else M)
    if op == "fluxdiff":  # one kernel per call: the step events time the launch
        kern_ms, kern_launches = t_total * 1e3, args.steps
        launches_per_step = 1
    peak, peak_src = measured_peak_gbs()
    alg_bytes = 2 * C * elem * local_cells  # per step-kernel launch (one partition per rank)
    kname = {"fused": {1: "k_sweep", 2: "k_step2d_ra",
                       3: "k_step3d_ra"}[D],
             "split": "k_sweep"}[args.kernel]
    if wl.get("order", 1) == 2:
        kname = {2: "k_step2d_o2", 3: "k_step2d_o2<3> (x-y) + k_zmarch2 (z)"}.get(D, "k_sweep2") \
            if (args.kernel == "fused" and args.layout == "soa") else "k_sweep2"
    if op == "fluxdiff":
        kname = ("k_fluxdiff_ra" if wl["dtype"] == "f32" else "k_fluxdiff_pt") \
            if (args.kernel == "fused" and D == 2 and args.layout == "soa") else "k_fluxdiff"
    per_launch_ms = kern_ms / max(kern_launches, 1)
    launches_per_step_kernel = max(1, kern_launches // max(5, min(args.steps, 20)))
    if args.kernel == "split" or D != 2:
        alg_bytes_launch = alg_bytes  # each sweep reads+writes the state once
    else:
        alg_bytes_launch = alg_bytes
    achieved = alg_bytes_launch / (per_launch_ms / 1e3) / 1e9
    if args.workload == "l256":
        traffic = ncu_traffic(f"{args.workload}_{wl['dtype']}_{args.layout}")
    elif op == "fluxdiff" and wl["dtype"] == "f64":
        traffic = ncu_traffic(f"{args.workload}_f64")
    else:
        traffic = ncu_traffic(f"{args.workload}_{args.kernel}")
    roof = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
            "peak_source": f"{peak_src} hbm_gbs (MEASURED_PEAKS.json copy bandwidth, burst)",
            "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
            "alg_bytes_per_launch": alg_bytes_launch, "launch_ms": per_launch_ms,
            "launches_per_step": launches_per_step_kernel,
            "frac_of_8TBs": achieved / 8000.0}
    if op == "step" and wl.get("order", 1) == 1:
        # the second ceiling of this path: floating-point issue.  Algorithmic FP
        # instructions per cell-step of the scheme as written in scheme.cuh (DESIGN.md
        # §6: 2-D 132, 3-D 240, 1-D 52; no tile recompute) against the measured issue
        # rate of tools/dp_microbench.cu (fp64 57.4, fp32 122.1 lanes/clk/SM at
        # 1.965 GHz on 148 SMs).
        ops = {1: 52, 2: 132, 3: 240}[D]
        lanes = 57.41 if elem == 8 else 122.11
        peak_g = lanes * 148 * 1.965
        ach_g = ops * local_cells / (per_launch_ms / 1e3) / 1e9 / \
            (D if args.kernel == "split" else 1)
        roof["fp_issue"] = {"ops_per_cell": ops, "achieved_gops": ach_g, "peak_gops": peak_g,
                            "frac": ach_g / peak_g,
                            "peak_source": "profiles/r1/dp_microbench.txt (measured)"}
    vs = None
    if op == "fluxdiff" and wl.get("paper_ms"):
        # paper Table 4 (V100, strided) time for the same pass: context, other hardware
        vs = wl["paper_ms"] / (t_total / args.steps * 1e3)
    line = {"metric": "Gcell/s (flux difference)" if op == "fluxdiff" else "Gcell-updates/s",
            "value": value, "unit": "Gcell/s" if op == "fluxdiff" else "Gcell-updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_total / args.steps * 1e3,
            "step_ms": {"min": min(step_list), "median": statistics.median(step_list),
                        "max": max(step_list), "n": len(step_list),
                        "how": "per-step CUDA events (max over ranks per step)"},
            "higher_is_better": True,
            "scaling": wl["scaling"], "vs_baseline": vs, "dtype": wl["dtype"],
            "data": "synthetic",
            "config": {"workload": wl["label"], "global_cells": gn, "parts": parts,
                       "kernel": args.kernel, "layout": args.layout,
                       "transport": args.transport if world > 1 else None,
                       "l2": "flushed between steps (256 MiB write), per-step CUDA events"
                             if flush is not None else "not flushed",
                       "timing": "sum of per-step CUDA events on the library stream, max over ranks",
                       "wall_s": wall, "dt": dt, "S0": S0, "op": op,
                       "cfl": {"loop": args.cfl_loop, "steps_per_run": M, "cfl": 0.9}
                       if op == "cfl" else None,
                       "paper_v100_ms": wl.get("paper_ms")},
            "roofline": roof, "gpu_launches": launches_per_step * args.steps,
            "halo": {"exposed_ms_per_step": exposed_ms if op == "step" else None,
                     "how": "per-step event time minus the step kernels' own event time "
                            "(profiled pass): halo pack/unpack, NCCL or P2P flag sync and "
                            "launch gaps; at N=1 only the launch gap + profiling events"},
            "clocks": clk.summary()}
    if e2e:
        line["e2e"] = e2e
    if op == "step" and args.workload == "2d1024" and world == 1:
        # configs[1] as a job: one rpl_advance(dt, 100) call from U0 (kernels back to
        # back, no flush).  The 67 MB working set stays in the 126 MB L2 -- reported
        # next to the flushed per-step headline, flagged as L2-resident.
        dom.set_state(U0)
        dom.advance(dt, 100)  # warm-up run
        dom.set_state(U0)
        r0 = torch.cuda.Event(enable_timing=True)
        r1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        r0.record(stream)
        dom.advance(dt, 100)
        r1.record(stream)
        torch.cuda.synchronize()
        dom.synchronize()
        run_ms = r0.elapsed_time(r1)
        line["run100"] = {"value": global_cells * 100 / (run_ms / 1e3) / 1e9,
                          "unit": "Gcell-updates/s", "ms_per_step": run_ms / 100,
                          "l2": "resident: 2 x 35 MB state < 126 MB L2, no flush inside the run",
                          "how": "one rpl_advance(dt, 100) call from U0, CUDA events on the "
                                 "library stream (BASELINE configs[1]: 100 steps on 1 B200)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(wl)
    if rank == 0:
        print(json.dumps(line), flush=True)
    dom.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
