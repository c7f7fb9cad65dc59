#!/usr/bin/env python
"""bench.py -- throughput of the split FORCE step (Ripple, arXiv 2104.08571) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--workload 2d1024|s512|w384|l256] [--kernel fused|split]

Metric (BASELINE.json): Gcell-updates/s = global interior cells x steps / time / 1e9,
plus the HBM-roofline fraction of the dominant kernel.

Default workload = BASELINE.json configs[2] (the headline): 3-D Euler, 512^3 cells,
fp64, SoA, shock-bubble data (workloads.shock_bubble), fixed dt = 0.4 dx / S0,
strong scaling (z-slabs at N > 1), with configs[3] (384^3 fp32 per GPU, weak, 2-D/3-D
blocks) and configs[1] (1024^2 fp64 per GPU, weak: the 2-D domain grows in x and y
and is split along y, the paper's setup P:1393-1402) as extra lines with their own
roofline.  L2 is flushed (256 MiB write + read) between timed steps and each step
is timed with its own CUDA events on the library's stream (flush excluded).  At N > 1
without torchrun the script relaunches itself under torch.distributed.run (one
process per GPU).

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
                  label="2-D Euler FORCE 6400x4000 fp64, y-split (paper strong 'small', P:1407)",
                  paper={"hardware": "8x V100-SXM2 16 GB (AWS p3, P:1130-1141)", "steps": 1000,
                         "speedup_8": 6.92, "efficiency_8_stated": 0.875,
                         "efficiency_8_from_speedup": 6.92 / 8,
                         "cite": "P:1404-1414 (sec. 8.2); formula P:1382"}),
    "p9600": dict(ndim=2, n=(9600, 6000), dtype="f64", scaling="strong",
                  label="2-D Euler FORCE 9600x6000 fp64, y-split (paper strong 'large', P:1408)",
                  paper={"hardware": "8x V100-SXM2 16 GB (AWS p3, P:1130-1141)", "steps": 1000,
                         "speedup_8": 7.32, "efficiency_8_stated": 0.915,
                         "efficiency_8_from_speedup": 7.32 / 8,
                         "cite": "P:1404-1414 (sec. 8.2); formula P:1382"}),
    "pweak": dict(ndim=2, n=(2560, 2500), dtype="f64", scaling="weak",
                  label="2-D Euler FORCE 6.4M cells/GPU fp64, y-split (paper weak, P:1393-1402)",
                  paper={"hardware": "8x V100-SXM2 16 GB (AWS p3, P:1130-1141)", "steps": 1000,
                         "weak_efficiency_8": "around 0.95",
                         "cite": "P:1399-1402, P:1503 (sec. 8.1); formula P:1378"}),
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


HEADLINE = "s512"            # BASELINE configs[2]: the metric's strong-scaling config
EXTRAS = ("w384", "2d1024")  # configs[3] (weak scaling), configs[1] (the 1-GPU 100-step job)


def _grow_xy(nranks):
    """2-D weak scaling as the paper runs it: the domain grows in x and
    y while it is split along y into nranks strips of the per-GPU size."""
    sx = 1
    while sx * sx * 2 <= nranks and nranks % (sx * 2) == 0:
        sx *= 2
    return sx, nranks // sx


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
        return [n[d] * parts[d] for d in range(D)], parts
    if D == 2:
        # y-split into nranks strips of n[0] x n[1] cells: global (n0 sx, n1 sy)
        sx, sy = _grow_xy(nranks)
        if (n[1] * sy) % nranks == 0:
            return [n[0] * sx, n[1] * sy], [1, nranks]
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
    """(dram bytes read+write per launch of the step kernel, source) from the committed
    ncu --set full summary (profiles/ncu_traffic.json, written by tools/ncu_summary.py
    with the capture file and its date), else (None, None)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            e = json.load(f).get(key)
    except Exception:
        return None, None
    if isinstance(e, dict):
        return e["bytes"], (f"ncu --set full capture {e.get('capture')} of {e.get('kernel')} "
                            f"({e.get('date')}), not this run")
    if e is not None:
        return e, "ncu --set full capture (round 1, profiles/r1/), not this run"
    return None, None


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _oracle_sample(wl, cap3d=128, cap2d=2048):
    """A bounded sample of the workload for the oracle: the same recipe on a sub-box."""
    import numpy as np

    import oracle
    import workloads as W
    D = wl["ndim"]
    n = list(wl["n"])
    if D == 3:
        n = [min(v, cap3d) for v in n]
    elif D == 2 and n[0] * n[1] > cap2d * cap2d:
        n = [cap2d, cap2d]
    dx = [1.0 / wl["n"][0]] * D
    U = W.shock_bubble(tuple(n), dx=dx)
    if wl["dtype"] == "f32":
        U = U.astype(np.float32)
    g = oracle.Grid(tuple(n), pad=wl.get("pad", 2), dx=dx, order=wl.get("order", 1))
    dt = 0.4 * dx[0] / oracle.max_wavespeed(g, U.astype(np.float64))
    return n, g, U, dt


def _oracle_run(wl, g, U, dt, k):
    """k units of the workload's op on the oracle (the same op the GPU arm times)."""
    import oracle
    op = wl.get("op", "step")
    if op == "fluxdiff":  # one flux-difference pass per unit (Table 4 kernel)
        for _ in range(k):
            oracle.flux_difference(g, U, dt)
    elif op == "cfl":  # cfl_steps CFL steps per unit (wavespeed pass + dt every step)
        oracle.run_cfl(g, U, 1e9, cfl=0.9, n_reduced=0, max_steps=k * wl.get("cfl_steps", 1))
    else:
        oracle.step(g, U, dt, k)


def _oracle_rate(wl, g, U, dt, threads, budget_s, cells):
    import oracle
    oracle.set_threads(threads)
    try:
        t0 = time.perf_counter()
        _oracle_run(wl, g, U, dt, 1)
        one = time.perf_counter() - t0
        k = max(1, min(1000, int(budget_s / max(one, 1e-6))))
        t0 = time.perf_counter()
        _oracle_run(wl, g, U, dt, k)
        el = time.perf_counter() - t0
    finally:
        oracle.set_threads(1)
    return cells * k * wl.get("cfl_steps", 1) / el / 1e9, k, el


def cpu_baseline(wl, budget_s=10.0):
    """The oracle as it stands (plain C; OpenMP over transverse lines, results identical
    for any thread count) on a bounded sample of the workload, at all host cores and at
    one thread."""
    import numpy as np
    n, g, U, dt = _oracle_sample(wl)
    cells = int(np.prod(n))
    cores = host_cores()
    v1, k1, e1 = _oracle_rate(wl, g, U, dt, 1, budget_s, cells)
    vn, kn, en = _oracle_rate(wl, g, U, dt, cores, budget_s, cells)
    op = wl.get("op", "step")
    unit = "Gcell/s" if op == "fluxdiff" else "Gcell-updates/s"
    what = {"fluxdiff": "flux-difference passes", "cfl": "CFL runs"}.get(op, "steps")
    return {"value": vn, "unit": unit, "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"{'x'.join(map(str, n))} sub-box of the same shock-bubble recipe, "
                      f"{wl['dtype']}{' order 2' if wl.get('order', 1) == 2 else ''}, {kn} {what} "
                      f"in {en:.1f} s on {cores} OpenMP threads (plain-C oracle)",
            "single_thread": {"value": v1, "cores": 1,
                              "sample": f"{k1} {what} in {e1:.1f} s"}}


def run_reference(args, wl):
    """--impl reference: the oracle on this arm's config and metric, on the host cores
    (rank 0 only; the other ranks exit without work)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    n, g, U, dt = _oracle_sample(wl, cap3d=96, cap2d=1024)
    cells = int(np.prod(n))
    cores = host_cores()
    oracle.set_threads(cores)
    try:
        for _ in range(args.warmup):
            _oracle_run(wl, g, U, dt, 1)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            _oracle_run(wl, g, U, dt, 1)
        el = time.perf_counter() - t0
    finally:
        oracle.set_threads(1)
    units = args.steps * wl.get("cfl_steps", 1)
    value = cells * units / el / 1e9
    op = wl.get("op", "step")
    unit = "Gcell/s" if op == "fluxdiff" else "Gcell-updates/s"
    full = n == list(wl["n"])
    sample = (f"{'x'.join(map(str, n))} {'(the full grid)' if full else 'sub-box of the workload'}"
              f" per step, op={op}, plain-C oracle on {cores} OpenMP threads ({cpu_model()})")
    line = {"impl": "reference", "metric": "Gcell/s (flux difference)" if op == "fluxdiff"
            else "Gcell-updates/s", "value": value,
            "unit": unit, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
            "higher_is_better": True, "scaling": wl["scaling"], "vs_baseline": None,
            "dtype": wl["dtype"], "data": "synthetic",
            "config": {"workload": wl["label"], "sample": sample},
            "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "oracle",
                             "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


def relaunch_torchrun(argv, n):
    """--gpus N > 1 without a torchrun environment: run this script under
    torch.distributed.run with N ranks (rank 0 prints the line)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
           str(n), "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


class Ctx:
    """Process / device plumbing shared by every workload of one bench run."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        # RPL_SHARE_DEVICE=1: every rank on cuda:0 (functional check of the N>1 path on
        # a 1-GPU box; timings are then meaningless: the processes time-slice one GPU)
        self.share = os.environ.get("RPL_SHARE_DEVICE") == "1"
        # torch.distributed over NCCL for the plumbing (ncclUniqueId broadcast, IPC-handle
        # all-gather, max-over-ranks timing); gloo only when all ranks share one GPU
        # (NCCL rejects two ranks on one device)
        self.backend = "gloo" if self.share else "nccl"
        if self.share and args.transport == "nccl":
            raise SystemExit("RPL_SHARE_DEVICE=1 needs --transport p2p (NCCL: one rank per GPU)")
        if self.world > 1:
            torch.cuda.set_device(0 if self.share else self.local_rank)
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local_rank))
            else:
                dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(0)
        self.dev = torch.cuda.current_device()
        # a real (non-default) stream shared by the library, the events and the L2 flush
        self.stream = torch.cuda.Stream()
        torch.cuda.set_stream(self.stream)
        self.flush = None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8,
                                                             device="cuda")
        self.flush_rd = None if args.no_flush else torch.ones(32 << 20, dtype=torch.float64,
                                                               device="cuda")
        self.flush_acc = torch.zeros((), dtype=torch.float64, device="cuda")

    def do_flush(self):
        # write 256 MiB (evicts the state from the 126 MB L2), then read another 256 MiB
        # so the L2 holds clean lines: the next step pays no write-backs of the flush
        if self.flush is not None:
            self.flush.fill_(1)
            self.flush_acc.add_(self.flush_rd.sum())

    def allmax(self, vals):
        """Element-wise max over ranks of a list of floats."""
        if self.world <= 1:
            return list(vals)
        t = self.torch.tensor(list(vals), dtype=self.torch.float64,
                              device="cuda" if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.cpu().tolist()

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()


def timed_loop(ctx, dom, step, nsteps, profile=False, sleep=True):
    """nsteps calls of step(), each bracketed by CUDA events on the library stream, L2
    flushed between calls (outside the events), barrier + synchronize on both sides.
    profile=True: the library also brackets every step-kernel launch (rpl_profile) and,
    multi-rank, every halo exchange (rpl_profile_halo).  Returns (per-step ms list,
    (kernel ms, launches), (halo ms, exchanges))."""
    torch = ctx.torch
    if profile:
        dom.profile(nsteps * 64)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(nsteps)]
    ctx.barrier()
    torch.cuda.synchronize()
    # GPU-side head start so the host queues the steps ahead of the GPU: the step
    # events then measure device time, not host launch latency
    if sleep:
        torch.cuda._sleep(200_000 * nsteps)
    for k in range(nsteps):
        ev[k][0].record(ctx.stream)
        step()
        ev[k][1].record(ctx.stream)
        ctx.do_flush()
    torch.cuda.synchronize()
    ctx.barrier()
    kern = dom.profile_read() if profile else (0.0, 0)
    halo = dom.profile_halo() if (profile and ctx.world > 1) else (0.0, 0)
    if profile:
        dom.profile(0)
    return [a.elapsed_time(b) for a, b in ev], kern, halo


def run_workload(ctx, args, name, steps, warmup, e2e_steps, headline):
    """Measure one workload; returns its JSON fields (value, timing, roofline, halo...)."""
    import numpy as np

    import paper_2104_08571_b200 as R
    import workloads as W
    wl = dict(WORKLOADS[name])
    if headline and args.dtype:
        wl["dtype"] = args.dtype
    world, rank = ctx.world, ctx.rank
    gn, parts = decomposition(wl, world)
    D = wl["ndim"]
    dx = [1.0 / wl["n"][0]] * D
    op = wl.get("op", "step")
    layout = args.layout if headline else "soa"
    kernel = args.kernel if headline else "fused"

    def make(transport):
        nccl_id = None
        if world > 1 and transport == "nccl":
            torch = ctx.torch
            idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if rank == 0:
                idt.copy_(torch.frombuffer(bytearray(R.nccl_unique_id()), dtype=torch.uint8))
            ctx.dist.broadcast(idt, 0)
            nccl_id = bytes(idt.cpu().numpy().tobytes())
        return R.Domain(gn, pad=wl.get("pad", 2), parts=parts, dtype=wl["dtype"], kernel=kernel,
                        dx=dx, layout=layout, nranks=world, rank=rank if world > 1 else 0,
                        nccl_id=nccl_id, device=ctx.dev, stream=ctx.stream.cuda_stream,
                        rows_per_chunk=args.rows,
                        transport=transport if world > 1 else "nccl", order=wl.get("order", 1))

    transport = args.transport
    dom = make(transport)
    if world > 1 and transport == "p2p":
        # P2P needs CUDA IPC + peer access between every pair of GPUs; if any rank cannot
        # attach, all ranks fall back to the NCCL transport (same arithmetic, bitwise)
        blobs = [None] * world
        ok = 1
        try:
            ctx.dist.all_gather_object(blobs, dom.p2p_export())
            dom.p2p_attach(blobs)
        except Exception as e:  # noqa: BLE001 -- reported, then the collective decision
            print(f"bench: rank {rank}: P2P attach failed ({e}); falling back to NCCL",
                  file=sys.stderr)
            ok = 0
        flag = ctx.torch.tensor([ok], dtype=ctx.torch.int32, device="cuda")
        ctx.dist.all_reduce(flag, op=ctx.dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            dom.close()
            transport = "nccl"
            dom = make(transport)
    box = (dom.lo, dom.hi)
    U0 = W.shock_bubble(tuple(gn), dx=dx, box=box)
    if wl["dtype"] == "f32":
        U0 = U0.astype(np.float32)
    dom.set_state(U0)
    S0 = dom.max_wavespeed()
    dt = 0.4 * min(dx) / S0
    local_n = [dom.box[d] for d in range(D)]
    local_cells = int(np.prod(local_n))
    global_cells = int(np.prod(gn))
    elem = 8 if wl["dtype"] == "f64" else 4
    C = D + 2
    M = wl.get("cfl_steps", 1)

    def run_cfl():
        # t_end far away: every run takes exactly M steps (the max_steps bound)
        if args.cfl_loop == "device":
            t, n = dom.advance_to(1e9, cfl=0.9, n_reduced=0, max_steps=M)
        else:
            n = dom.advance_cfl(1e9, cfl=0.9, n_reduced=0, max_steps=M)
        assert n == M, n

    def step():
        if op == "fluxdiff":
            dom.flux_difference(dt)
        elif op == "cfl":
            run_cfl()
        else:
            dom.advance(dt, 1)

    for _ in range(warmup):
        step()
        ctx.do_flush()
    ctx.torch.cuda.synchronize()
    launches_per_step = dom.launches_per_step
    wall0 = time.perf_counter()
    with Clocks(ctx.dev) as clk:
        step_list, _, _ = timed_loop(ctx, dom, step, steps, sleep=op != "cfl")  # the headline
    wall = time.perf_counter() - wall0
    # the step kernel's own launch time for the roofline and the event-timed halo
    # (separate, profiled pass: the event pairs cost a few us per launch)
    n_prof = max(5, min(steps, 20))
    prof_list, (kern_ms, kern_launches), (halo_ms, n_exch) = timed_loop(
        ctx, dom, step, n_prof, profile=True, sleep=op != "cfl")
    step_list = ctx.allmax(step_list)     # per step: max over ranks
    t_total = sum(step_list) / 1e3
    dom.synchronize()  # surfaces any domain error of the timed steps
    kname = dom.kernel_name("fluxdiff" if op == "fluxdiff" else "step")

    # ---- exposed halo per step, multi-rank only
    halo = {"exposed_ms_per_step": None, "event_ms_per_step": None, "differential_ms_per_step": None,
            "note": "N=1: one partition, no halo exchange (the ghost images are written by the "
                    "step kernel itself)"}
    if world > 1 and op == "step":
        ev_ms = ctx.allmax([halo_ms / n_prof])[0]
        # differential: the same local partition alone on this GPU (nranks 1, exchange
        # disabled: physical boundaries instead of halos), timed the same way
        solo = R.Domain(local_n, pad=wl.get("pad", 2), dtype=wl["dtype"], kernel=kernel, dx=dx,
                        layout=layout, device=ctx.dev, stream=ctx.stream.cuda_stream,
                        rows_per_chunk=args.rows, order=wl.get("order", 1))
        solo.set_state(np.ascontiguousarray(U0))

        def solo_step():
            solo.advance(dt, 1)
        for _ in range(warmup):
            solo_step()
            ctx.do_flush()
        solo_list, _, _ = timed_loop(ctx, solo, solo_step, steps)
        solo.close()
        t_solo = ctx.allmax([sum(solo_list) / len(solo_list)])[0]
        diff = t_total * 1e3 / steps - t_solo
        halo = {"exposed_ms_per_step": max(ev_ms, 0.0), "event_ms_per_step": ev_ms,
                "differential_ms_per_step": diff, "solo_ms_per_step": t_solo,
                "exchanges_per_step": n_exch / n_prof,
                "how": "event: t(halo ready) - t(interior done) per exchange, library events "
                       "around the exchange (rpl_profile_halo), max over ranks; differential: "
                       "step time at N ranks - step time of the same local partition alone "
                       "(nranks 1, exchange disabled), max over ranks"}

    # ---- e2e through the public API with host buffers (pinned), copies timed
    e2e = None
    if e2e_steps > 0:
        torch = ctx.torch
        tdt = torch.float64 if elem == 8 else torch.float32
        h_in = torch.empty(C * local_cells, dtype=tdt, pin_memory=True)
        h_out = torch.empty(C * local_cells, dtype=tdt, pin_memory=True)
        h_in.numpy()[:] = np.ascontiguousarray(np.moveaxis(U0, -1, 0)).ravel()
        dom.get_state_ptr(h_out.data_ptr())
        torch.cuda.synchronize()
        ctx.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        for _ in range(e2e_steps):
            dom.set_state_ptr(h_in.data_ptr())
            if op == "fluxdiff":
                dom.flux_difference(dt)
                N_get_fd(dom, h_out.data_ptr())
            else:
                step()
                dom.get_state_ptr(h_out.data_ptr())
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        te = ctx.allmax([e0.elapsed_time(e1) / 1e3])[0]
        nb = C * local_cells * elem
        e2e = {"value": global_cells * M * e2e_steps / te / 1e9, "unit": "Gcell-updates/s",
               "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb, "steps": e2e_steps,
               "path": "rpl_set_state(pinned host) + rpl_advance(dt,1) + rpl_get_state(pinned host)"}

    value = global_cells * M * steps / t_total / 1e9
    if op == "cfl":
        # device loop: M step launches + the initial wavespeed pass; host loop: a
        # wavespeed pass before every step
        launches_per_step = M * launches_per_step + (1 if args.cfl_loop == "device" else M)
    if op == "fluxdiff":  # one kernel per call: the step events time the launch
        kern_ms, kern_launches = sum(prof_list), n_prof
        launches_per_step = 1
    peak, peak_src = measured_peak_gbs()
    per_launch_ms = kern_ms / max(kern_launches, 1)
    launches_per_step_kernel = max(1, kern_launches // n_prof)
    alg_bytes_launch = 2 * C * elem * local_cells  # read U^n once, write U^{n+1} once
    achieved = alg_bytes_launch / (per_launch_ms / 1e3) / 1e9
    if name == "l256":
        tkey = f"{name}_{wl['dtype']}_{layout}"
    elif op == "fluxdiff" and wl["dtype"] == "f64":
        tkey = f"{name}_f64"
    else:
        tkey = f"{name}_{kernel}"
    traffic, traffic_src = ncu_traffic(tkey)
    roof = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
            "peak_source": f"{peak_src} hbm_gbs (MEASURED_PEAKS.json copy bandwidth, burst)",
            "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
            "traffic_source": traffic_src,
            "alg_bytes_per_launch": alg_bytes_launch,
            "alg_bytes_how": f"2 x C x s x local interior cells = 2 x {C} x {elem} B x "
                             f"{local_cells}",
            "launch_ms": per_launch_ms, "launches_per_step": launches_per_step_kernel,
            "launch_timing": "CUDA event pair around every step-kernel launch on the "
                             "library stream (rpl_profile), profiled pass of "
                             f"{n_prof} steps",
            "frac_of_8TBs": achieved / 8000.0}
    if op == "step" and wl.get("order", 1) == 1:
        # the second ceiling of this path: floating-point issue.  Algorithmic FP
        # operations per cell-step of the scheme as written in scheme.cuh (cell_ab /
        # face_psi / psi_update, reading A1 and 6: 9D + 35 per sweep, i.e.
        # 2-D 106, 3-D 186, 1-D 44; no tile recompute) against the measured lane rate
        # of tools/dp_microbench.cu (fp64 57.4, fp32 122.1 lanes/clk/SM at 1.965 GHz
        # on 148 SMs).
        ops = {1: 44, 2: 106, 3: 186}[D]
        lanes = 57.41 if elem == 8 else 122.11
        peak_g = lanes * 148 * 1.965
        ach_g = ops * local_cells / (per_launch_ms / 1e3) / 1e9 / \
            (D if kernel == "split" else 1)
        roof["fp_issue"] = {"ops_per_cell": ops, "achieved_gops": ach_g, "peak_gops": peak_g,
                            "frac": ach_g / peak_g,
                            "peak_source": "profiles/r1/dp_microbench.txt (measured)"}
    vs = None
    if op == "fluxdiff" and wl.get("paper_ms"):
        # paper Table 4 (V100, strided) time for the same pass: context, other hardware
        vs = wl["paper_ms"] / (t_total / steps * 1e3)
    out = {"metric": "Gcell/s (flux difference)" if op == "fluxdiff" else "Gcell-updates/s",
           "value": value, "unit": "Gcell/s" if op == "fluxdiff" else "Gcell-updates/s",
           "ms_per_step": t_total / steps * 1e3,
           "step_ms": {"min": min(step_list), "median": statistics.median(step_list),
                       "max": max(step_list), "n": len(step_list),
                       "how": "per-step CUDA events (max over ranks per step)"},
           "scaling": wl["scaling"], "vs_baseline": vs, "dtype": wl["dtype"],
           "config": {"workload": wl["label"], "global_cells": gn, "parts": parts,
                      "kernel": kernel, "layout": layout,
                      "transport": transport if world > 1 else None,
                      "l2": "flushed between steps (256 MiB write + 256 MiB read), per-step "
                            "CUDA events" if ctx.flush is not None else "not flushed",
                      "timing": "sum of per-step CUDA events on the library stream, max over "
                                "ranks per step",
                      "wall_s": wall, "dt": dt, "S0": S0, "op": op,
                      "cfl": {"loop": args.cfl_loop, "steps_per_run": M, "cfl": 0.9}
                      if op == "cfl" else None,
                      "paper_v100_ms": wl.get("paper_ms"),
                      "paper_context": wl.get("paper")},
           "roofline": roof, "gpu_launches": launches_per_step * steps,
           "halo": halo, "clocks": clk.summary()}
    if e2e:
        out["e2e"] = e2e
    if op == "step" and name == "2d1024" and world == 1:
        # configs[1] as a job: one rpl_advance(dt, 100) call from U0 (kernels back to
        # back, no flush).  The 67 MB working set stays in the 126 MB L2 -- reported
        # next to the flushed per-step number, flagged as L2-resident.
        torch = ctx.torch
        dom.set_state(U0)
        dom.advance(dt, 100)  # warm-up run
        dom.set_state(U0)
        r0 = torch.cuda.Event(enable_timing=True)
        r1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        r0.record(ctx.stream)
        dom.advance(dt, 100)
        r1.record(ctx.stream)
        torch.cuda.synchronize()
        dom.synchronize()
        run_ms = r0.elapsed_time(r1)
        out["run100"] = {"value": global_cells * 100 / (run_ms / 1e3) / 1e9,
                         "unit": "Gcell-updates/s", "ms_per_step": run_ms / 100,
                         "l2": "resident: 2 x 35 MB state < 126 MB L2, no flush inside the run",
                         "how": "one rpl_advance(dt, 100) call from U0, CUDA events on the "
                                "library stream (BASELINE configs[1]: 100 steps on 1 B200)"}
    dom.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=HEADLINE, choices=sorted(WORKLOADS))
    ap.add_argument("--extras", default="auto",
                    help="extra workloads measured in the same run, each with its own "
                         "roofline: 'auto' (= w384,2d1024 with the default headline), "
                         "'none', or a comma list")
    ap.add_argument("--extra-steps", type=int, default=20)
    ap.add_argument("--cfl-loop", default="device", choices=["device", "host"],
                    help="cfl workloads: rpl_advance_to (device-side dt) or rpl_advance_cfl "
                         "(host loop: wavespeed pass + sync every step)")
    ap.add_argument("--kernel", default="fused", choices=["fused", "split"])
    ap.add_argument("--dtype", default=None, choices=["f32", "f64"],
                    help="override the workload's dtype (configs[4] runs both)")
    ap.add_argument("--layout", default="soa", choices=["soa", "aos"],
                    help="HBM layout of the conserved-state struct (BASELINE configs[4])")
    ap.add_argument("--rows", type=int, default=0, help="z-planes per 3-D chunk (0 = auto)")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="halo transport between ranks (N > 1): P2P = step kernels store halos "
                         "into the neighbour's buffer over NVLink (CUDA IPC); NCCL = pack + "
                         "ncclSend/Recv + unpack")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_torchrun(sys.argv[1:], args.gpus)
    wl = dict(WORKLOADS[args.workload])
    if args.dtype:
        wl["dtype"] = args.dtype
    if args.impl == "reference":
        return run_reference(args, wl)
    if args.extras == "auto":
        extras = list(EXTRAS) if args.workload == HEADLINE else []
    elif args.extras == "none":
        extras = []
    else:
        extras = [e for e in args.extras.split(",") if e]
    for e in extras:
        if e not in WORKLOADS:
            raise SystemExit(f"unknown extra workload {e}")

    ctx = Ctx(args)
    head = run_workload(ctx, args, args.workload, args.steps, args.warmup, args.e2e_steps, True)
    line = {"metric": head.pop("metric"), "value": head.pop("value"), "unit": head.pop("unit"),
            "n_gpus": ctx.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": head.pop("ms_per_step"), "higher_is_better": True}
    line.update({"scaling": head.pop("scaling"), "vs_baseline": head.pop("vs_baseline"),
                 "dtype": head.pop("dtype"), "data": "synthetic"})
    line.update(head)
    if extras:
        line["extra"] = {}
        for e in extras:
            x = run_workload(ctx, args, e, args.extra_steps, 3, 0, False)
            x["steps"] = args.extra_steps
            line["extra"][e] = x
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(wl)
    if ctx.rank == 0:
        print(json.dumps(line), flush=True)
    if ctx.world > 1:
        ctx.dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
