#!/usr/bin/env python
"""Benchmark of the divergence-uncertainty hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config {0..4}] [--impl {ours,reference}]
    python bench.py --workload {lcp,gradient,fit,ingest,redsea}   # SURVEY 8f rows, 1 GPU

Default workload = BASELINE.json config 3 (the metric's "1/2/4/8 B200" config):
3D analytic divergence mean + sigma + P(div>0) + P(div<0) on a 512^3 fp32
grid, z-slab sharded over N GPUs (strong scaling; NCCL halo exchange of the
w edge planes overlapped with the interior planes).  One "step" = one pass of
the hot path over the whole grid with inputs resident in HBM.

Prints ONE JSON line (rank 0).  Keys beyond the base contract:
  roofline      dominant kernel: algorithmic bytes per launch / its average
                CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the oracle restatement of the reference on this box's cores
  e2e           the same metric through the host-buffer C-ABI entry point
                (pinned host buffers, H2D + D2H inside the timed region)
  gpu_launches  our kernel launches inside the timed region
  clocks        NVML SM clock / throttle reasons sampled during the timed region

``--impl reference`` times the reference's CPU implementation on this box's
host cores, rank 0 only, on the same fixed sample as the cpu_baseline leg
(oracle/cpu_baseline.cpu_leg): the unmodified reference package
(baseline/_ref, its own pip install) for the 2D configs, the oracle
restatement for the 3D configs (the reference has no 3D code).

``--gpus N`` outside torchrun launches the N ranks itself (one process per
GPU, torch.distributed.run on 127.0.0.1, NCCL_DEBUG=INFO).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ERR = None   # the device validation word of the timed calls (int32 CUDA tensor)


def validation_note():
    """Read the validation word once after the timed loop; raise like the
    reference would on bad inputs, else describe the check for the JSON line."""
    from paper_2510_01190_b200.device import raise_for_bits

    bits = int(ERR.item())
    raise_for_bits(bits)
    return "on: kernels validate every input (non-finite, sigma < 0) into a device word, read once after the timed loop (clean)"


METRIC = "grid points/sec (analytic div mean+var+prob) and % HBM roofline at 1/2/4/8 B200"
UNIT = "grid points/s"


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def committed_traffic(key):
    """dram bytes per launch from the committed ncu --set full capture, or None."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(key)
    except Exception:
        return None


class ClockSampler:
    """NVML SM clock + clocks-event reasons, polled every ~2 ms in a thread."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x1: "gpu_idle"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], 0, False
        self.stop_evt = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self.stop_evt.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop_evt.set()
            self.th.join()
            try:  # one more sample right at the end of the timed region
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            except Exception:
                pass

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": names, "n_samples": len(self.samples)}


class L2Flush:
    """Between timed launches: write a 256 MB buffer (> the 126 MB L2), then
    read a second one, so the inputs are evicted AND the flush's own dirty
    lines are written back before the timed kernel starts (otherwise their
    write-back would steal HBM bandwidth inside the timed region)."""

    NOTE = "flushed between steps (256 MB write, then 256 MB read to drain dirty lines)"

    def __init__(self, torch):
        self.w = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        self.r = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
        self.i64 = torch.int64

    def __call__(self):
        self.w.zero_()
        return self.r.sum(dtype=self.i64)


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(args):
    """The reference's own CPU implementation of the path on this box's host
    cores (oracle/cpu_baseline.cpu_leg: the unmodified reference from
    baseline/_ref for the 2D configs, the oracle restatement for the 3D ones
    that have no reference code), the SAME fixed sample the repo arm's
    cpu_baseline leg times, each step one call.  Rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return  # rank 0 alone runs the CPU reference
    from oracle import cpu_baseline as cb

    cid = args.config
    threads = os.cpu_count() or 1
    steps, warm = args.steps, args.warmup
    work, units, unit, sample, kind = cb.cpu_leg(cid, threads)
    par = True
    if cid in (0, 1):   # the faster of the reference's threaded and serial paths
        t0 = time.perf_counter(); work(True); work(True); tp = time.perf_counter() - t0
        t0 = time.perf_counter(); work(False); work(False); ts = time.perf_counter() - t0
        par = tp <= ts
    times = []
    for it in range(warm + steps):
        t0 = time.perf_counter()
        work(par) if cid in (0, 1) else work()
        if it >= warm:
            times.append(time.perf_counter() - t0)
    mean_s = sum(times) / len(times)
    value = units / mean_s
    cores = threads if par else 1
    line = {
        "impl": "reference", "metric": METRIC if cid != 2 else "vertex-samples/sec (Monte Carlo divergence mean+std)",
        "value": value, "unit": unit, "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": mean_s * 1e3, "higher_is_better": True,
        "scaling": "strong" if cid == 3 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": f"config{cid} (bounded CPU sample)"},
        "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": kind,
                         "sample": sample + ("" if par else "; serial path (faster than threaded)")},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def maybe_spawn(args) -> bool:
    """``--gpus N`` without a torchrun environment: launch N ranks ourselves
    (torch.distributed.run, one process per GPU, rendezvous on 127.0.0.1) and
    exit with their status.  Under torchrun the world size must equal N."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None:
        if int(env_world) != args.gpus:
            raise SystemExit(f"bench.py: WORLD_SIZE={env_world} but --gpus {args.gpus}")
        return False
    if args.gpus <= 1:
        return False
    if os.environ.get("DIVUQ_BENCH_ONE_DEVICE") != "1" and not args.plumbing_check:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible")
    import socket
    import subprocess

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd, env=env))


def plumbing_check(args):
    """--plumbing-check: the multi-rank launch path without GPU work (CPU
    test): every rank joins a gloo group, the ranks all-reduce their count,
    rank 0 prints the JSON skeleton with n_gpus = the world size."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.ones(1)
    if world > 1:
        dist.all_reduce(t)
    print(f"rank {rank}/{world}: process group up ({'gloo' if world > 1 else 'none'})", file=sys.stderr,
          flush=True)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "n_gpus": world, "ranks_seen": int(t.item()),
                          "plumbing_check": True}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# SURVEY 8f "next" rows: LCP, gradient prologue, DIVUQ1 ingest (1 GPU lines)
# ---------------------------------------------------------------------------

def run_next(args):
    """One JSON line for a widened row (not a BASELINE config; same keys)."""
    import torch

    import __graft_entry__

    __graft_entry__.build()
    from paper_2510_01190_b200 import configs, device as dev, io as dio
    from paper_2510_01190_b200._lib import lib

    torch.cuda.set_device(0)
    global ERR
    ERR = torch.zeros(1, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()
    peak, peak_src = measured_peak()
    ev_pairs = []

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    flush = L2Flush(torch)
    wl = args.workload
    if wl == "lcp":
        nx = ny = 4096
        model = configs.host_model2d(nx, ny, 24, 105)
        dm = [torch.from_numpy(a).cuda() for a in model]
        o = dev.propagate2d(*dm, nx, ny, 1.0, 1.0, 0.0, outputs=("mu", "sigma"))
        mu, sg = o["mu"], o["sigma"]
        units = (nx - 1) * (ny - 1)
        bpu = 8 * 2 * nx * ny / units + 8  # mu, sigma read once per vertex + one fp64 out per cell
        unit = "cells/s"
        metric = "level-crossing probability cells/sec (lcp.py:80-100), fp64"
        workload = "lcp: per-cell P(div field crosses 0) on a 4096^2 fp64 divergence (mu, sigma) field"

        def step():
            dev.lcp2d(mu, sg, nx, ny, 0.0, check=ERR)

        hm, hs = mu.cpu().pin_memory(), sg.cpu().pin_memory()
        hout = torch.empty(units, dtype=torch.float64).pin_memory()

        def e2e_call():
            st = lib.divuq_host_lcp2d_f64(hm.data_ptr(), hs.data_ptr(), nx, ny, 0.0,
                                          hout.data_ptr(), 0)
            assert st == 0, st

        h2d, d2h = 16 * nx * ny, 8 * units
        mu_h, sg_h = hm.numpy()[: 1024 * 1024], hs.numpy()[: 1024 * 1024]
        from oracle import ref2d

        cpu_thunk = (lambda: ref2d.lcp(mu_h, sg_h, 1024, 1024, 0.0), 1023 * 1023, 1)
        cpu_sample = "numpy restatement of lcp() on a 1024x1024 corner of the field, 1 thread"
        dtype = "f64"
    elif wl == "lcpfused":   # propagate -> lcp in one pass (fused)
        nx = ny = 4096
        model = configs.host_model2d(nx, ny, 24, 105)
        dm = [torch.from_numpy(a).cuda() for a in model]
        outs = {"lcp": torch.empty((nx - 1) * (ny - 1), dtype=torch.float64, device="cuda")}
        units = (nx - 1) * (ny - 1)
        bpu = 8 * 4 * nx * ny / units + 8  # (mu_u, mu_v, s_u, s_v) read once per vertex + one fp64 out per cell
        unit = "cells/s"
        metric = ("level-crossing probability cells/sec of the divergence field, fused "
                  "propagate_divergence -> lcp (divergence.py:48-70 + lcp.py:80-100), fp64")
        workload = ("lcpfused: P(div crosses 0) per cell straight from the 4096^2 fp64 Gaussian (u, v) "
                    "model, one kernel (moments not written)")

        def step():
            dev.propagate_lcp2d(*dm, nx, ny, 1.0, 1.0, 0.0, moments=False, out=outs, check=ERR)

        k2o = {k: torch.empty(nx * ny, dtype=torch.float64, device="cuda") for k in ("mu", "sigma")}

        def composed():
            dev.propagate2d(*dm, nx, ny, 1.0, 1.0, 0.0, outputs=("mu", "sigma"), out=k2o, check=ERR)
            dev.lcp2d(k2o["mu"], k2o["sigma"], nx, ny, 0.0, check=ERR)

        hin = [torch.from_numpy(a).pin_memory() for a in model]
        hout = torch.empty(units, dtype=torch.float64).pin_memory()

        def e2e_call():
            st = lib.divuq_host_propagate_lcp2d_f64(*(t.data_ptr() for t in hin), nx, ny, 1.0, 1.0, 0.0,
                                                    None, None, hout.data_ptr(), 0)
            assert st == 0, st

        h2d, d2h = 32 * nx * ny, 8 * units
        sub = [a[: 1024 * 1024] for a in model]
        from oracle import ref2d

        def cpu_work():
            mu_d, sg_d = ref2d.propagate2d(*sub, 1024, 1024, 1.0, 1.0)
            ref2d.lcp(mu_d, sg_d, 1024, 1024, 0.0)

        cpu_thunk = (cpu_work, 1023 * 1023, 1)
        cpu_sample = "numpy restatement of propagate_divergence + lcp() on a 1024x1024 corner, 1 thread"
        dtype = "f64"
    elif wl == "gradient":
        nx = ny = 1024
        m = 20
        mem = configs.config1_members(nx, ny, m, 101).double()
        out = torch.empty_like(mem)
        units = m * nx * ny
        bpu = 32  # u, v in + gx, gy out, fp64, per member-vertex
        unit = "member-vertices/s"
        metric = "velocity-magnitude-gradient member-vertices/sec (gaussian.py:48-66), fp64"
        workload = "gradient: gradient_ensemble of the config-1 ensemble (M=20, 1024^2), fp64"

        def step():
            dev.gradient_ensemble2d(mem, nx, ny, 1.0, 1.0, out=out, check=ERR)

        hin = mem.cpu().pin_memory()
        hout = torch.empty_like(hin).pin_memory()

        def e2e_call():
            st = lib.divuq_host_gradient_ensemble2d_f64(hin.data_ptr(), m, nx, ny, 1.0, 1.0,
                                                        hout.data_ptr(), 0)
            assert st == 0, st

        h2d = d2h = 16 * units
        sub = hin.numpy()[:4, :, : 256 * 1024]
        from oracle import ref2d

        cpu_thunk = (lambda: ref2d.gradient_ensemble(sub, 1024, 256, 1.0, 1.0), 4 * 256 * 1024, 1)
        cpu_sample = "numpy restatement (hypot + reference stencil), 4 members x 1024x256, 1 thread"
        dtype = "f64"
    elif wl == "redsea":   # K6: the Red Sea pipeline fused (gradient prologue -> K3)
        nx = ny = 1024
        m = 20
        mem = configs.config1_members(nx, ny, m, 101)
        outs = {k: torch.empty(nx * ny, dtype=torch.float32, device="cuda") for k in dev.ALL_OUTPUTS}
        units = nx * ny
        bpu = 2 * m * 4 + 4 * 4   # M members x (u, v) fp32 in, four fp32 maps out
        unit = "grid points/s"
        metric = ("grid points/sec, velocity-magnitude-gradient ensemble -> divergence mean+var+"
                  "P(div>0)+P(div<0) (gaussian.py:48-66 + 35-45, divergence.py, lcp.py:48-68), fp32")
        workload = ("redsea: fused |v| -> gradient -> moments -> divergence -> tails on the config-1 "
                    "velocity ensemble (M=20, 1024^2), fp32, one kernel")

        def step():
            dev.gradient_ensemble_divergence2d(mem, nx, ny, 1.0, 1.0, 0.0, out=outs, check=ERR)

        # the same chain unfused (gradient ensemble written + re-read), for the record
        grad = torch.empty_like(mem)

        def composed():
            dev.gradient_ensemble2d(mem, nx, ny, 1.0, 1.0, out=grad, check=ERR)
            dev.ensemble_divergence2d(grad, nx, ny, 1.0, 1.0, 0.0, out=outs, check=ERR)

        hin = mem.cpu().pin_memory()
        hout = [torch.empty(units, dtype=torch.float32).pin_memory() for _ in range(4)]

        def e2e_call():
            st = lib.divuq_host_gradient_ensemble_divergence2d_f32(
                hin.data_ptr(), m, nx, ny, 1.0, 1.0, 0.0, *(t.data_ptr() for t in hout), None, None, 0)
            assert st == 0, st

        h2d, d2h = m * 2 * 4 * units, 16 * units
        import numpy as np

        sub = hin.numpy()[:, :, : 1024 * 64].astype(np.float64)
        from oracle import ref2d

        def cpu_work():
            g = ref2d.gradient_ensemble(sub, 1024, 64, 1.0, 1.0)
            mu_f, sg_f = ref2d.fit_moments(g)
            mu_d, sg_d = ref2d.propagate2d(mu_f[0], mu_f[1], sg_f[0], sg_f[1], 1024, 64, 1.0, 1.0)
            ref2d.source_probability(mu_d, sg_d, 0.0)
            ref2d.sink_probability(mu_d, sg_d, 0.0)

        cpu_thunk = (cpu_work, 1024 * 64, 1)
        cpu_sample = ("numpy restatement of gradient_ensemble -> fit_gaussian -> propagate -> both "
                      "tails on a 1024x64 strip (all 20 members), fp64, 1 thread")
        dtype = "f32"
    elif wl == "fit":   # K1: the drop-in fit_gaussian (gaussian.py:35-45), fp64 bitwise
        nx = ny = 1024
        m = 20
        mem = configs.config1_members(nx, ny, m, 101).double()
        mu_o = torch.empty((2, nx * ny), dtype=torch.float64, device="cuda")
        sg_o = torch.empty_like(mu_o)
        units = nx * ny
        bpu = 2 * m * 8 + 2 * 2 * 8   # M members x (u, v) in, (mu, sigma) x (u, v) out, fp64
        unit = "grid points/s"
        metric = "ensemble fit_gaussian grid points/sec (gaussian.py:35-45), fp64 (numpy bitwise)"
        workload = "fit: fit_gaussian of the config-1 ensemble (M=20, 1024^2) in fp64"

        def step():
            dev.fit_moments(mem, out=(mu_o, sg_o), check=ERR)

        hin = mem.cpu().pin_memory()
        hmu = torch.empty((2, nx * ny), dtype=torch.float64).pin_memory()
        hsg = torch.empty_like(hmu).pin_memory()

        def e2e_call():
            st = lib.divuq_host_fit_gaussian_f64(hin.data_ptr(), m, 2, nx * ny, hmu.data_ptr(),
                                                 hsg.data_ptr(), 0)
            assert st == 0, st

        h2d, d2h = m * 2 * 8 * units, 4 * 8 * units
        sub = hin.numpy()[:, :, : 1024 * 64]
        from oracle import ref2d

        cpu_thunk = (lambda: ref2d.fit_moments(sub), 1024 * 64, 1)
        cpu_sample = "numpy restatement of fit_gaussian (the reference's numpy calls), 1024x64, 1 thread"
        dtype = "f64"
    else:  # ingest: DIVUQ1 file -> HBM -> fused fit/propagate/tails (the CLI's pipeline)
        import tempfile

        nx = ny = 1024
        m = 20
        mem = configs.config1_members(nx, ny, m, 101)
        host = mem.cpu().numpy()
        tmpdir = tempfile.mkdtemp(prefix="divuq_bench_")
        path = os.path.join(tmpdir, "config1.duq")
        st = lib.divuq_divuq1_write_f32(os.fsencode(path), nx, ny, 1.0, 1.0, m, host.ctypes.data)
        assert st == 0, st
        units = nx * ny
        file_bytes = host.nbytes
        unit = "grid points/s"
        metric = "DIVUQ1 file -> P(div>0) maps grid points/sec (io.py:58-93 + config 1 pipeline)"
        workload = ("ingest: DIVUQ1 file (config-1 ensemble M=20 1024^2, 168 MB, page-cache "
                    "resident) -> pinned staging -> HBM -> fused fit/propagate/tails, fp32")
        outs = {k: torch.empty(units, dtype=torch.float32, device="cuda") for k in ("mu", "sigma", "p_src")}

        def step():
            _, x = dio.load_ensemble_device(path)
            dev.ensemble_divergence2d(x, nx, ny, 1.0, 1.0, 0.0, outputs=("mu", "sigma", "p_src"),
                                      out=outs, check=ERR)

        e2e_call = None
        h2d, d2h = file_bytes, 0
        from oracle import divuq1, ref2d

        def cpu_work():
            (_, _, _, _), planes = divuq1.read_members(path)
            mu_f, sg_f = ref2d.fit_moments(planes)
            mu_d, sg_d = ref2d.propagate2d(mu_f[0], mu_f[1], sg_f[0], sg_f[1], nx, ny, 1.0, 1.0)
            ref2d.source_probability(mu_d, sg_d, 0.0)

        cpu_thunk = (cpu_work, units, 1)
        cpu_sample = "oracle reader + fit_gaussian + propagate + P(div>0) on the same file, fp64, 1 thread"
        dtype = "f32"

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = 1 if wl != "ingest" else 1
    with ClockSampler(0) as clocks:
        if wl == "ingest":  # host work inside the step: wall clock around synchronized steps
            t0 = time.perf_counter()
            for _ in range(args.steps):
                step()
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) * 1e3 / args.steps
            ev_ms = None
        else:
            for _ in range(args.steps):
                flush()  # L2 flush; outside the kernel events
                a = ev()
                step()
                ev_pairs.append((a, ev()))
            torch.cuda.synchronize()
            ev_ms = [a.elapsed_time(b) for a, b in ev_pairs]
            ms = sum(ev_ms) / len(ev_ms)
    value = units / (ms * 1e-3)
    if wl == "ingest":
        # the bound is the host->device link: measure pinned H2D of the same bytes
        src = torch.from_numpy(host).pin_memory()
        dst = torch.empty_like(mem)
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        a = ev()
        for _ in range(5):
            dst.copy_(src, non_blocking=True)
        b = ev()
        torch.cuda.synchronize()
        h2d_gbs = file_bytes * 5 / (a.elapsed_time(b) * 1e-3) / 1e9
        achieved = file_bytes / (ms * 1e-3) / 1e9
        roofline = {"bound": "pcie (host->device)", "achieved": achieved, "peak": h2d_gbs,
                    "unit": "GB/s", "frac": achieved / h2d_gbs, "traffic": None,
                    "peak_source": "pinned cudaMemcpy H2D of the same 168 MB, measured in this run",
                    "bytes_per_step": file_bytes}
        e2e = {"value": value, "unit": unit, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": ms, "path": "io.load_ensemble_device (divuq_divuq1_ingest_f32) + K3 2D"}
    else:
        achieved = bpu * units / (ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": committed_traffic(wl),
                    "bytes_per_unit": bpu, "units_per_launch": units, "avg_launch_ms": ms,
                    "peak_source": peak_src}
        if wl in ("redsea", "lcpfused"):   # the unfused chain on the same input, same protocol
            if wl == "redsea":
                roofline["note"] = ("same byte count as config 1 (+4 B/pt): its small-problem floor, "
                                    "36.1 us for a perfectly coalesced stream (profiles/r01/bwbench.txt), "
                                    "applies")
            comp_ms = []
            for _ in range(args.steps):
                flush()
                a = ev()
                composed()
                b = ev()
                comp_ms.append((a, b))
            torch.cuda.synchronize()
            roofline["unfused_chain_ms"] = sum(a.elapsed_time(b) for a, b in comp_ms) / len(comp_ms)
        e2e_call()
        reps = 3
        t0 = time.perf_counter()
        for _ in range(reps):
            e2e_call()
        e2e_s = (time.perf_counter() - t0) / reps
        e2e = {"value": units / e2e_s, "unit": unit, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3}
    cpu = None
    if not args.no_cpu:
        from oracle import cpu_baseline as cb

        v, thr, runs = cb.rate(cpu_thunk, seconds=8.0)
        cpu = {"value": v, "unit": unit, "cores": thr, "kind": "port",
               "sample": cpu_sample + f", {runs} runs"}
    if wl == "ingest":
        os.remove(path)
        os.rmdir(tmpdir)
    line = {
        "metric": metric, "value": value, "unit": unit, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": dtype, "data": "synthetic (seeded generator)",
        "config": {"workload": workload, "parallelism": "replicas x1",
                   "l2": L2Flush.NOTE if wl != "ingest" else "n/a (host-bound)",
                   "validation": validation_note()},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps, "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=3, choices=(0, 1, 2, 3, 4))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fp64", action="store_true", help="skip config 3's fp64 side measurement")
    ap.add_argument("--planes-per-gpu", type=int, default=128, help="config 4 slab depth")
    ap.add_argument("--exchange", default="p2p", choices=("p2p", "nccl"),
                    help="z-slab halo exchange for configs 3/4 at N>1: peer memory read in "
                         "place by the kernels (p2p) or NCCL send/recv overlapped with the interior")
    ap.add_argument("--plumbing-check", action="store_true",
                    help="multi-rank launch/rendezvous only (no GPU work): CPU test of --gpus N")
    ap.add_argument("--workload", default=None,
                    choices=("lcp", "lcpfused", "gradient", "ingest", "fit", "redsea"),
                    help="a SURVEY 8f row instead of a BASELINE config (1 GPU, ours only)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "ours" and args.workload is None:
        maybe_spawn(args)      # exits after the ranks finish when it launched them
    if args.plumbing_check:
        plumbing_check(args)
        return
    if args.workload is not None:
        if args.impl == "reference" or int(os.environ.get("RANK", "0")) != 0:
            return
        run_next(args)
        return

    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # DIVUQ_BENCH_ONE_DEVICE=1: dry run of the sharded orchestration with every
    # rank on cuda:0 over gloo (the p2p slab path never makes a rank wait on
    # another's kernels, so this is safe); its numbers are NOT multi-GPU numbers
    one_device = os.environ.get("DIVUQ_BENCH_ONE_DEVICE") == "1"
    if one_device:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    global ERR
    ERR = torch.zeros(1, dtype=torch.int32, device="cuda")
    import __graft_entry__

    if rank == 0:
        __graft_entry__.build()
    if world > 1:
        dist.barrier()
    from paper_2510_01190_b200 import configs, device as dev
    from paper_2510_01190_b200._lib import lib
    from paper_2510_01190_b200 import shard
    from paper_2510_01190_b200.shard import SlabStep

    cfg = configs.CONFIGS[args.config]
    stream = torch.cuda.current_stream()
    kernel_events = []  # (start, end) of the dominant launch per step

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    exchange_used = args.exchange
    if args.config == 3:
        nx, ny, nz = cfg.nx, cfg.ny, cfg.nz
        step = SlabStep(nx, ny, nz, rank, world, device="cuda", exchange=args.exchange)
        fields = configs.config3_slab(step.z0, step.nzl, nx, ny, nz, seed=cfg.seed)
        n_local = nx * ny * step.nzl
        out = {k: torch.empty(n_local, dtype=torch.float32, device="cuda") for k in dev.ALL_OUTPUTS}
        plane = nx * ny
        mu_w, s_w = fields[2], fields[5]
        shard.ensure_p2p(step, {"mu_w": mu_w, "s_w": s_w})   # falls back to NCCL on every rank
        exchange_used = step.exchange
        total_pts = nx * ny * nz
        scaling = "strong"

        def edges():
            return ((mu_w[:plane], s_w[:plane]), (mu_w[-plane:], s_w[-plane:]))

        def compute(k_range, lo, hi, timed):
            dominant = (k_range[1] - k_range[0]) > 1 or step.nzl == 1
            e0 = ev() if timed and dominant else None
            dev.propagate3d(*fields, nx, ny, step.nzl, 1.0, 1.0, 1.0, cfg.t, z0=step.z0,
                            nz_global=nz, halo_lo=step.halo_lo, halo_hi=step.halo_hi,
                            k_range=k_range, out=out, check=ERR)
            if e0 is not None:
                kernel_events.append((e0, ev(), (k_range[1] - k_range[0]) * plane))
            return 1

        def one_step(timed):
            if step.exchange == "p2p" and world > 1:   # one launch, halos read over NVLink
                e0 = ev() if timed else None
                # inputs are immutable during the loop and mapped once (ensure_p2p +
                # the barrier before timing): no per-step collective or fence
                n = shard.propagate3d_step(step, fields, out, 1.0, 1.0, 1.0, cfg.t, check=ERR,
                                           sync_inputs=False, fence=False, remap=False)
                if timed:
                    kernel_events.append((e0, ev(), step.nzl * plane))
                return n
            return step.run(edges, lambda kr, lo, hi: compute(kr, lo, hi, timed))

        bpp = cfg.bytes_per_point
        workload = ("config3: 3D analytic divergence mean+sigma+P(div>0)+P(div<0), fp32, "
                    f"512^3, z-slab x{world}")
    elif args.config == 4:
        nx, ny = cfg.nx, cfg.ny
        nz = args.planes_per_gpu * world
        step = SlabStep(nx, ny, nz, rank, world, n_arrays=3, device="cuda", exchange=args.exchange)
        members = configs.config4_slab(step.z0, step.nzl, nx, ny, nz, cfg.members, cfg.seed)
        shard.ensure_p2p(step, {"members": members})
        exchange_used = step.exchange
        n_local = nx * ny * step.nzl
        out = {k: torch.empty(n_local, dtype=torch.float32, device="cuda") for k in dev.ALL_OUTPUTS}
        total_pts = nx * ny * nz
        scaling = "weak"

        def edges():
            first = dev.w_moments_plane(members, nx, ny, step.nzl, 0, check=ERR)
            last = dev.w_moments_plane(members, nx, ny, step.nzl, step.nzl - 1, check=ERR)
            return first, last

        def compute(k_range, lo, hi, timed):
            dominant = (k_range[1] - k_range[0]) > 1
            e0 = ev() if timed and dominant else None
            dev.ensemble_divergence3d(members, nx, ny, step.nzl, 1.0, 1.0, 1.0, cfg.t, z0=step.z0,
                                      nz_global=nz, halo_lo=step.halo_lo, halo_hi=step.halo_hi,
                                      k_range=k_range, out=out, check=ERR)
            if e0 is not None:
                kernel_events.append((e0, ev(), (k_range[1] - k_range[0]) * nx * ny))
            return 1

        def one_step(timed):
            if step.exchange == "p2p" and world > 1:   # neighbours' edge moments read over NVLink
                e0 = ev() if timed else None           # (whole step timed: conservative roofline)
                n = shard.ensemble3d_step(step, members, out, 1.0, 1.0, 1.0, cfg.t, check=ERR,
                                          sync_inputs=False, fence=False, remap=False)
                if timed:
                    kernel_events.append((e0, ev(), step.nzl * nx * ny))
                return n
            n = step.run(edges, lambda kr, lo, hi: compute(kr, lo, hi, timed))
            return n + (2 if world > 1 else 0)

        bpp = cfg.bytes_per_point
        workload = (f"config4 slab: fused ensemble (M=16) -> moments -> divergence -> P(div>0.1), "
                    f"P(div<-0.1), fp32, 1024x1024x{args.planes_per_gpu} per GPU "
                    f"(N=8 -> the full 1024^3 config 4)")
    elif args.config == 0:  # 2D analytic fp64 128^2 (L2-resident, launch-bound): replicas only
        nx, ny = cfg.nx, cfg.ny
        host_model = configs.config0_model()
        model = [torch.from_numpy(a).cuda() for a in host_model]
        n_local = nx * ny
        out = {k: torch.empty(n_local, dtype=torch.float64, device="cuda") for k in dev.ALL_OUTPUTS}
        total_pts = nx * ny * world
        scaling = "weak"
        flush = L2Flush(torch)

        def one_step(timed):
            if timed:
                flush()  # L2 flush between steps; outside the kernel events
            e0 = ev() if timed else None
            dev.propagate2d(*model, nx, ny, 1.0, 1.0, cfg.t, out=out, check=ERR)
            if timed:
                kernel_events.append((e0, ev(), nx * ny))
            return 1

        bpp = cfg.bytes_per_point
        workload = "config0: 2D analytic divergence mean+sigma+P(div>0)+P(div<0), fp64, 128^2"
    elif args.config == 2:  # Monte Carlo fp64 256^2 x 2000 samples: replicas only
        nx, ny = cfg.nx, cfg.ny
        host_model = configs.config2_model()
        model = [torch.from_numpy(a).cuda() for a in host_model]
        n_local = nx * ny
        mean = torch.empty(n_local, dtype=torch.float64, device="cuda")
        std = torch.empty_like(mean)
        total_pts = nx * ny * cfg.n_samples * world
        scaling = "weak"

        def one_step(timed):
            e0 = ev() if timed else None
            dev.mc_divergence2d(*model, nx, ny, 1.0, 1.0, cfg.n_samples, 2024, out=(mean, std),
                                check=ERR)
            if timed:
                kernel_events.append((e0, ev(), nx * ny))
            return 2

        bpp = cfg.bytes_per_point
        workload = "config2: 2D Monte Carlo divergence mean/std, fp64, 256^2, N=2000, Philox4x32-10"
    else:  # config 1: 2D fused ensemble, replicas only
        nx, ny = cfg.nx, cfg.ny
        members = configs.config1_members(nx, ny, cfg.members, cfg.seed)
        n_local = nx * ny
        out = {k: torch.empty(n_local, dtype=torch.float32, device="cuda")
               for k in ("mu", "sigma", "p_src")}
        total_pts = nx * ny * world
        scaling = "weak"
        flush = L2Flush(torch)

        def one_step(timed):
            if timed:
                flush()  # L2 flush (inputs 168 MB are ~L2-sized); outside the kernel events
            e0 = ev() if timed else None
            dev.ensemble_divergence2d(members, nx, ny, 1.0, 1.0, cfg.t, outputs=("mu", "sigma", "p_src"),
                                      out=out, check=ERR)
            if timed:
                kernel_events.append((e0, ev(), nx * ny))
            return 1

        bpp = cfg.bytes_per_point
        workload = "config1: 2D fused ensemble M=20 -> moments -> divergence -> P(div>0), fp32, 1024^2"

    # correctness guard on the real inputs before timing (validation word)
    torch.cuda.synchronize()
    if world > 1:   # every slab is written before any peer reads it in place (p2p)
        dist.barrier()

    for _ in range(args.warmup):
        one_step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = 0
    with ClockSampler(local) as clocks:
        t_start = ev()
        for _ in range(args.steps):
            launches += one_step(True)
        t_end = ev()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    elapsed_ms = t_start.elapsed_time(t_end)
    if args.config in (0, 1):  # flushes excluded: sum of kernel intervals
        elapsed_ms = sum(a.elapsed_time(b) for a, b, _ in kernel_events)
    if world > 1:
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    value = total_pts / (ms_per_step * 1e-3)

    # roofline of the dominant kernel (rank 0's launches)
    k_ms = [a.elapsed_time(b) for a, b, _ in kernel_events]
    k_pts = kernel_events[0][2] if kernel_events else n_local
    avg_k_s = (sum(k_ms) / len(k_ms)) * 1e-3 if k_ms else ms_per_step * 1e-3
    peak, peak_src = measured_peak()
    achieved = bpp * k_pts / avg_k_s / 1e9
    traffic = committed_traffic(f"config{args.config}")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "bytes_per_point": bpp, "points_per_launch": k_pts,
                "avg_launch_ms": avg_k_s * 1e3, "peak_source": peak_src}
    if args.config == 2:  # fp64-ALU bound: the HBM fraction is not the bound that matters
        # fp64 flops per vertex-sample of mc_chunk_kernel, counted from the ncu
        # SASS source page (predicated-on thread instructions: DFMA x2 + DMUL +
        # DADD; round 2 after the table sin/cos: 92.3 -- round 1 counted 108.7)
        flops_vs = 92.3
        fp64_peak = 148 * 64 * 2 * 1.965e9 / 1e12   # vector fp64 FMA pipe, TFLOP/s at max clock
        vs_launch = cfg.n_samples * nx * ny
        achieved_tf = flops_vs * vs_launch / avg_k_s / 1e12
        roofline = {"bound": "fp64 (CUDA-core FMA pipe; no tensor-core work)", "achieved": achieved_tf,
                    "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved_tf / fp64_peak,
                    "traffic": traffic, "flops_per_vertex_sample": flops_vs,
                    "peak_source": "148 SMs x 64 fp64 FMA/clk x 2 x 1.965 GHz (nominal; ncu: fp64 pipe ~49 % busy)",
                    "note": ("Philox + Box-Muller per vertex-sample; HBM traffic is ~48 B/vertex; the "
                             "kernel is issue-bound: 207 thread instructions per vertex-sample (ncu), "
                             "0.73 ms at 100 % of the issue slots"),
                    "avg_launch_ms": avg_k_s * 1e3}
    elif args.config == 0:
        roofline["note"] = "0.9 MB working set: launch/latency-bound, L2 flushed between steps"
    elif args.config == 1:
        roofline["note"] = ("small-problem floor: a perfectly coalesced 40-read/3-write float4 stream of "
                            "the same 172 MB, timed the same way (L2 evicted, one launch), takes 36.1 us "
                            "= 5.0 TB/s (tools/bwbench, profiles/r01/bwbench.txt)")

    # the same config-3 workload in fp64 (the reference's precision), next to
    # the fp32 headline: single-GPU launches of the fp64 K2, same protocol
    fp64_variant = None
    if args.config == 3 and world == 1 and not args.no_fp64:
        f64 = [f.double() for f in fields]
        o64 = {k: torch.empty(n_local, dtype=torch.float64, device="cuda") for k in dev.ALL_OUTPUTS}
        for _ in range(3):
            dev.propagate3d(*f64, nx, ny, nz, 1.0, 1.0, 1.0, cfg.t, out=o64, check=ERR)
        pairs = []
        for _ in range(10):
            a = ev()
            dev.propagate3d(*f64, nx, ny, nz, 1.0, 1.0, 1.0, cfg.t, out=o64, check=ERR)
            pairs.append((a, ev()))
        torch.cuda.synchronize()
        ms64 = sum(a.elapsed_time(b) for a, b in pairs) / len(pairs)
        bpp64 = 6 * 8 + 4 * 8
        ach64 = bpp64 * n_local / (ms64 * 1e-3) / 1e9
        fp64_variant = {"dtype": "f64", "ms_per_step": ms64, "value": total_pts / (ms64 * 1e-3),
                        "unit": UNIT, "roofline": {"bound": "hbm", "achieved": ach64, "peak": peak,
                                                   "unit": "GB/s", "frac": ach64 / peak,
                                                   "bytes_per_point": bpp64},
                        "note": "k2_tma_kernel<double>: the reference's fp64 arithmetic, bitwise to the "
                                "reference order; 10 launches, inputs 6.4 GB (> L2)"}
        del f64, o64
        torch.cuda.empty_cache()

    # e2e through the host-buffer C ABI (pinned host buffers, copies timed)
    e2e = None
    if not args.no_e2e and args.config == 3:
        host_in = [f.cpu().pin_memory() for f in fields]
        host_out = [torch.empty(n_local, dtype=torch.float32).pin_memory() for _ in range(4)]
        g_nz = step.nzl  # each rank pushes its own slab through the host entry point
        chunk = 16       # tools/e2e_chunk_probe.py: 8/16/32/64/128 -> 67.8/67.3/68.9/72.5/80.7 ms

        def e2e_call():
            st = lib.divuq_host_propagate3d_f32(
                *(t.data_ptr() for t in host_in), nx, ny, g_nz, 1.0, 1.0, 1.0, cfg.t,
                *(t.data_ptr() for t in host_out), chunk, local)
            if st != 0:
                raise RuntimeError(f"host pipeline status {st}")

        e2e_call()
        if world > 1:
            dist.barrier()
        reps = 3
        t0 = time.perf_counter()
        for _ in range(reps):
            e2e_call()
        e2e_s = (time.perf_counter() - t0) / reps
        if world > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        h2d = 4 * 6 * n_local   # every field byte crosses PCIe once (halos read from HBM)
        e2e = {"value": total_pts / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d * world,
               "d2h_bytes_per_step": 16 * n_local * world, "ms_per_step": e2e_s * 1e3,
               "path": "divuq_host_propagate3d_f32 (pinned host buffers, 3-stream z-chunk pipeline)"}
    elif not args.no_e2e and args.config == 4:
        # each rank pushes its slab from pinned host memory through the host
        # entry; bounded so all ranks' pinned copies fit in 40% of host RAM
        plane = nx * ny
        plane_b = cfg.members * 3 * plane * 4
        ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
        e_planes = max(2, min(step.nzl, int(0.4 * ram) // (world * plane_b)))
        ez0, ez1 = step.z0, step.z0 + e_planes
        del members   # make room in HBM for the pipeline's staging sets
        torch.cuda.empty_cache()
        host_mem = torch.empty((cfg.members, 3, e_planes * plane), dtype=torch.float32, pin_memory=True)
        for z in range(0, e_planes, 8):   # generate on the device, 8 planes at a time
            k = min(8, e_planes - z)
            host_mem[:, :, z * plane:(z + k) * plane].copy_(
                configs.config4_slab(ez0 + z, k, nx, ny, nz, cfg.members, cfg.seed))
        ghost = {}
        for side, zg in (("lo", ez0 - 1), ("hi", ez1)):
            if 0 <= zg < nz:
                ghost[side] = configs.config4_slab(zg, 1, nx, ny, nz, cfg.members, cfg.seed)[:, 2].cpu()
        host_out = [torch.empty(e_planes * plane, dtype=torch.float32, pin_memory=True)
                    for _ in range(4)]

        def e2e_call():
            st = lib.divuq_host_ensemble_divergence3d_f32(
                host_mem.data_ptr(), cfg.members, nx, ny, e_planes, ez0, nz,
                ghost["lo"].data_ptr() if "lo" in ghost else None,
                ghost["hi"].data_ptr() if "hi" in ghost else None, plane, 1.0, 1.0, 1.0, cfg.t,
                *(t.data_ptr() for t in host_out), 0, local)
            if st != 0:
                raise RuntimeError(f"host entry status {st}")

        e2e_call()
        if world > 1:
            dist.barrier()
        reps = 3
        t0 = time.perf_counter()
        for _ in range(reps):
            e2e_call()
        e2e_s = (time.perf_counter() - t0) / reps
        if world > 1:
            t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e_pts = world * e_planes * plane
        h2d = host_mem.numel() * 4 + sum(g.numel() * 4 for g in ghost.values())
        e2e = {"value": e_pts / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d * world,
               "d2h_bytes_per_step": 16 * e_planes * plane * world, "ms_per_step": e2e_s * 1e3,
               "planes_per_gpu": e_planes,
               "path": "divuq_host_ensemble_divergence3d_f32 (pinned host members, 3-stream z-chunk "
                       "pipeline, each member byte over PCIe once)"}
    elif not args.no_e2e and args.config in (0, 2):
        host_in = [torch.from_numpy(a).pin_memory() for a in host_model]
        nouts = 4 if args.config == 0 else 2
        host_out = [torch.empty(n_local, dtype=torch.float64).pin_memory() for _ in range(nouts)]

        def e2e_call():
            if args.config == 0:
                st = lib.divuq_host_propagate2d_f64(*(t.data_ptr() for t in host_in), nx, ny, 1.0, 1.0,
                                                    cfg.t, *(t.data_ptr() for t in host_out), local)
            else:
                st = lib.divuq_host_mc_divergence2d_f64(*(t.data_ptr() for t in host_in), nx, ny, 1.0,
                                                        1.0, cfg.n_samples, 2024,
                                                        *(t.data_ptr() for t in host_out), local)
            if st != 0:
                raise RuntimeError(f"host entry status {st}")

        e2e_call()
        reps = 20 if args.config == 0 else 5
        t0 = time.perf_counter()
        for _ in range(reps):
            e2e_call()
        e2e_s = (time.perf_counter() - t0) / reps
        e2e = {"value": total_pts / e2e_s, "unit": UNIT if args.config == 0 else "vertex-samples/s",
               "h2d_bytes_per_step": 32 * n_local, "d2h_bytes_per_step": 8 * nouts * n_local,
               "ms_per_step": e2e_s * 1e3}
    elif not args.no_e2e and args.config == 1:
        import numpy as np

        host_mem = members.cpu().pin_memory()
        host_out = [torch.empty(n_local, dtype=torch.float32).pin_memory() for _ in range(3)]

        def e2e_call():
            st = lib.divuq_host_ensemble_divergence2d_f32(
                host_mem.data_ptr(), cfg.members, nx, ny, 1.0, 1.0, cfg.t,
                *(t.data_ptr() for t in host_out), None, None, None, local)
            if st != 0:
                raise RuntimeError(f"host entry status {st}")

        e2e_call()
        reps = 5
        t0 = time.perf_counter()
        for _ in range(reps):
            e2e_call()
        e2e_s = (time.perf_counter() - t0) / reps
        e2e = {"value": total_pts / e2e_s, "unit": UNIT, "h2d_bytes_per_step": host_mem.numel() * 4,
               "d2h_bytes_per_step": 12 * n_local, "ms_per_step": e2e_s * 1e3}
        _ = np

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import cpu_baseline as cb

        cpu = cb.time_leg(args.config, seconds=10.0)   # the reference arm's exact sample

    unit = "vertex-samples/s" if args.config == 2 else UNIT
    line = {
        "metric": METRIC if args.config != 2 else "vertex-samples/sec (Monte Carlo divergence mean+std)",
        "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64" if args.config in (0, 2) else "f32",
        "data": "synthetic (seeded generator, BASELINE.json config recipe)",
        "config": {"workload": workload, "grid_points": total_pts, "t": cfg.t,
                   "parallelism": f"z-slab x{world}" if args.config in (3, 4) else f"replicas x{world}",
                   "exchange": (("peer memory (CUDA IPC over NVLink), read in place by the kernels"
                                 if exchange_used == "p2p" else "NCCL send/recv overlapped with the interior")
                                + ("" if exchange_used == args.exchange else
                                   " (fallback: peer mapping failed on some rank)")
                                if args.config in (3, 4) and world > 1 else None),
                   **({"dry_run": "DIVUQ_BENCH_ONE_DEVICE=1: every rank on cuda:0 over gloo "
                                  "(orchestration check, not a multi-GPU number)"}
                      if one_device and world > 1 else {}),
                   "validation": validation_note(),
                   "l2": (L2Flush.NOTE if args.config in (0, 1) else
                          "inputs larger than L2 (126 MB); no flush" if args.config in (3, 4) else
                          "compute-bound; 2 MB model stays in L2")},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clocks.summary(),
    }
    if fp64_variant is not None:
        line["fp64_variant"] = fp64_variant
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
