#!/usr/bin/env python
"""Benchmark: 2D 5-point heat stencil (f32) over annotated, chunked distributed arrays.

Workload (BASELINE.json configs[1]): a 65536 x 65536 f32 grid, row-block stencil
distribution (halo [1, 0]) over N GPUs, one distributed `heat2d` launch per step:
planning (annotation -> regions -> tasks) + executor + halo exchange + kernel. Inputs are
resident in HBM (2 x 16 GiB, far larger than the 126 MB L2, so no flush is needed).

Reports (one JSON line, rank 0):
  value     cell-updates/s over K timed steps, CUDA events (all streams joined), max over ranks
  e2e       same metric through the public API with HOST buffers: per step, upload the grid
            from pinned memory, run `e2e_iters` heat iterations, read the grid back; steps
            pipelined with mt_array_write_async / mt_array_read_async over three array sets
            (N > 1: each rank moves its own chunk box); wall clock, max over ranks; the
            synchronous figure is reported beside it
  roofline  heat2d kernel: 8 algorithmic bytes per cell update / its average duration (CUDA
            events on the launching stream) vs MEASURED_PEAKS.json hbm_gbs
  clocks    nvidia-smi SM clocks and throttle reasons sampled during the timed region
  cpu_baseline  the reference CPU executor (oracle/_ref, the unmodified reference compiled from
            its sources) running the same kernel on a bounded row sample, all host threads
  N = 1 only: contraction (C3, tcgen05 bf16 32768^3), reductions (C4 histogram / k-means),
            small_grid (C1, 4096^2 in 4 chunks, with the reference on the same grid),
            out_of_core (C5 analog: spill tier against the pinned-link bound)

`--impl reference` times the reference CPU executor as the main arm (rank 0 only).
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

from ctypes import c_int as C_INT  # noqa: E402

METRIC = "stencil cell-updates/s + matmul TFLOP/s at 1/2/4/8 B200; % roofline; vs CPU ref"
ANN = "global [i, j] => read in[i-1:i+1, j-1:j+1], write out[i,j]"
ALPHA = 0.1
BYTES_PER_CELL = 8  # one f32 read + one f32 write per cell update


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(kernel_file: str, rows: int, cols: int):
    """dram read+write bytes per launch from the newest committed `ncu --set full` capture of
    this kernel (profiles/round*/<kernel_file>), when it was taken on the same grid."""
    import glob
    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "round*", kernel_file))):
        try:
            with open(path) as f:
                s = json.load(f)
        except Exception:
            continue
        if s.get("algorithmic_bytes_per_launch") == BYTES_PER_CELL * rows * cols:
            best = (s["traffic_bytes_per_launch"], os.path.relpath(path, ROOT))
    return best


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def barrier_max(value: float, ws: int) -> float:
    if ws == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def setup_heat(ctx, rows, cols, n_parts, block=(16, 16), strip=0):
    """Two f32 arrays in a row-block stencil distribution (halo [1, 0]), one chunk per device.
    With `strip` > 0 every device's rows become three superblocks (top strip, interior, bottom
    strip) so the interior, which reads no halo row, overlaps the halo exchange (
    region-precise dependencies make it independent of the incoming rows)."""
    from paper_2202_05549_b200 import Arr, Superblock
    devs = ctx.devices
    dist = lambda: ctx.dist.stencil([rows, cols], [rows // n_parts, cols], [1, 0], devs)  # noqa: E731
    a = ctx.create_array([rows, cols], "f32", dist(), 0)
    b = ctx.create_array([rows, cols], "f32", dist(), 0)
    work = ctx.dist.block_work([rows, cols], list(block), [rows // n_parts, cols], devs)
    if strip > 0:
        rb, sb, cb = rows // n_parts // block[0], strip // block[0], (cols + block[1] - 1) // block[1]
        work = []
        for i, d in enumerate(devs):
            b0, b1 = i * rb, (i + 1) * rb
            for lo, hi in ((b0, b0 + sb), (b0 + sb, b1 - sb), (b1 - sb, b1)):
                work.append(Superblock((lo, 0), (hi, cb), d))
    ctx.launch("ramp2d_f32", [rows, cols], list(block), work, [rows, cols, 1000, 0.0, 1.0, Arr(a)], "global [i, j] => write out[i,j]")
    ctx.flush()
    return a, b, work


def sample_rows(want: int, devices: int, block: int = 16) -> int:
    """rows of the CPU sample: a whole number of 16-row blocks per chunk, one chunk per device
    thread, as close to `want` as that allows (block_work_dist needs superblock extents that
    are multiples of the block, distribution.cpp:110-134)"""
    per = devices * block
    return per * max(1, round(want / per))


def host_cpu() -> dict:
    """the CPU model and thread counts the CPU baselines ran on"""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        affinity = len(os.sched_getaffinity(0))
    except AttributeError:
        affinity = os.cpu_count()
    return {"model": model, "nproc": affinity, "cpu_count": os.cpu_count()}


# One sampling protocol for the heat2d CPU baseline, shared by the main arm's cpu_baseline and
# `--impl reference`: a CPU_ROWS-row band of the full-width grid, one chunk (and device thread)
# per host thread, CPU_WARMUP untimed launches, then timed launches in the same context. The
# reference pipelines consecutive launches across chunks, so its rate climbs over
# the first few launches; timing after the warm-up gives the steady-state rate either arm sees.
CPU_ROWS, CPU_WARMUP, CPU_ITERS = 512, 10, 60


def cpu_reference_rate(rows, cols, iters, devices, bounds_check=True, warmup=CPU_WARMUP) -> tuple[float, float]:
    """Reference CPU executor (oracle/_ref) on a rows x cols sample: (cell-updates/s, seconds of
    the timed launches). bounds_check: the reference's array_view index checks (memory.hpp:54,
    default on)."""
    import oracle
    from paper_2202_05549_b200 import Arr
    ref = oracle.reference()
    toggle = getattr(ref.dll, "mr_set_bounds_check", None)
    if toggle is not None:
        toggle(C_INT(1 if bounds_check else 0))
    elif not bounds_check:
        raise RuntimeError("reference build lacks mr_set_bounds_check")
    ctx = oracle.reference_context(workers=1, devices=devices, execute=True)
    a, b, work = setup_heat(ctx, rows, cols, devices)

    def run(n):
        nonlocal a, b
        for _ in range(n):
            ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, ALPHA, Arr(b), Arr(a)], ANN)
            ctx.flush()
            a, b = b, a
        ctx.synchronize()

    run(warmup)
    t0 = time.perf_counter()
    run(iters)
    dt = time.perf_counter() - t0
    ctx.close()
    if toggle is not None:
        toggle(C_INT(1))
    return rows * cols * iters / dt, dt


def cpu_heat_baseline(cols, rows_total, want_rows=CPU_ROWS, steps=CPU_ITERS, warmup=CPU_WARMUP) -> dict:
    """the heat2d CPU baseline: the `--impl reference` arm itself, run as a fresh subprocess with
    the driver-style flags (so both numbers come from one protocol in the same kind of process:
    no GPU context, clock sampler or pinned host tier beside it), plus its sensitivity to the
    sample height (half the rows)"""
    import subprocess

    def arm(rows, bounds="on"):
        env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT")}
        cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference", "--rows", str(rows_total), "--cols", str(cols),
               "--cpu-rows", str(rows), "--steps", str(steps), "--warmup", str(warmup), "--cpu-bounds-check", bounds]
        r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600)
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        if r.returncode != 0 or not lines:
            raise RuntimeError(f"reference arm failed (rc {r.returncode}): {r.stderr[-300:]}")
        return json.loads(lines[-1])

    full = arm(want_rows)
    half = arm(want_rows // 2)
    cb = full["cpu_baseline"]
    out = {"value": full["value"], "unit": "cell-updates/s", "cores": cb["cores"], "kind": "reference",
           "sample": cb["sample"] + f" ({full['ms_per_step'] * steps / 1e3:.1f} s); the `--impl reference` protocol, run as a subprocess",
           "bounds_check": "on (the reference default, memory.hpp:54)", "host": cb.get("host"),
           "sensitivity": {"rows": half["config"]["rows"], "value": half["value"], "ratio": half["value"] / full["value"]}}
    try:  # the reference with its array_view bounds checks off as well
        off = arm(want_rows, "off")
        out["bounds_check_off"] = {"value": off["value"], "ratio": off["value"] / full["value"]}
    except Exception as e:  # noqa: BLE001
        out["bounds_check_off"] = {"unavailable": str(e)}
    return out


def cpu_matmul_baseline(sizes=(1024, 2048)) -> dict:
    """the reference `matmul` kernel (kernels.cpp:167-193: scalar f32 dot in l order) on the
    reference CPU executor with every host thread: A and C row blocks, B replicated (the
    replicated-input form of C3), inputs the C3 ramp patterns; FLOP/s = 2 n^3 / launch time.
    At the smallest size every element is checked against an fp64 product of the same inputs."""
    import numpy as np

    import oracle
    from paper_2202_05549_b200 import Arr
    threads = oracle.reference().host_threads()
    dv = max(1, min(threads, 64))
    runs = []
    for n in sizes:
        ctx = oracle.reference_context(workers=1, devices=dv, execute=True)
        devs = ctx.devices
        per = (n + dv - 1) // dv
        per = (per + 15) // 16 * 16
        A = ctx.create_array([n, n], "f32", ctx.dist.row([n, n], per, devs), 0)
        B = ctx.create_array([n, n], "f32", ctx.dist.replicated([n, n], devs), 0)
        Cm = ctx.create_array([n, n], "f32", ctx.dist.row([n, n], per, devs), 0)
        w = ctx.dist.block_work([n, n], [16, 16], [per, n], devs)
        ctx.launch("ramp2d_f32", [n, n], [16, 16], w, [n, n, 1000, 0.0, 1.0, Arr(A)], "global [i, j] => write out[i,j]")
        ctx.launch("ramp2d_f32", [n, n], [16, 16], ctx.dist.block_work([n, n], [16, 16], [n, n], devs[:1]), [n, n, 997, 0.0, 1.0, Arr(B)],
                   "global [i, j] => write out[i,j]")
        ctx.synchronize()
        t0 = time.perf_counter()
        ctx.launch("matmul", [n, n], [16, 16], w, [n, n, n, Arr(Cm), Arr(A), Arr(B)], "global [i, j] => write C[i,j], read A[i,:], read B[:,j]")
        ctx.synchronize()
        dt = time.perf_counter() - t0
        r = {"n": n, "value": 2.0 * n ** 3 / dt / 1e12, "seconds": dt}
        if n == min(sizes):
            c = ctx.read(Cm).astype(np.float64)
            want = ctx.read(A).astype(np.float64) @ ctx.read(B).astype(np.float64)
            r["max_rel_err_vs_fp64_all_elements"] = float(np.max(np.abs(c - want) / np.abs(want)))
        ctx.close()
        runs.append(r)
    best = max(runs, key=lambda r: r["value"])
    return {"value": best["value"], "unit": "TFLOP/s", "cores": dv, "kind": "reference",
            "sample": "reference `matmul` kernel (f32, kernels.cpp:167-193) at " + ", ".join(f"{r['n']}^3 ({r['seconds']:.1f} s)" for r in runs)
                      + f", 1 worker x {dv} device threads; value = the faster size",
            "sizes": runs, "host": host_cpu()}


def cpu_ooc_baseline(rows=2048, cols=8192, iters=4) -> dict:
    """the reference's out-of-core path (memory.cpp:245-377) at a reduced size: heat2d over two
    rows x cols f32 arrays in chunk_rows-row chunks, with every device's capacity a quarter of its
    working set (acceptance c4's squeeze), all host threads; cell-updates/s over timed launches
    after one warm-up launch, and the reference's own eviction counts"""
    import json as _json

    import oracle
    from paper_2202_05549_b200 import Arr
    threads = oracle.reference().host_threads()
    dv = max(1, min(threads, 64))
    # eight chunks per device: one task's footprint (its input chunk with halo rows plus its
    # output chunk) must fit the quarter capacity, which the reference checks (memory.cpp:278-287)
    chunk_rows = max(16, rows // (8 * dv) // 16 * 16)
    dv = max(1, min(dv, rows // chunk_rows // 8))
    per_dev_ws = 2 * rows * cols * 4 // dv
    cap = per_dev_ws // 4
    ctx = oracle.reference_context(workers=1, devices=dv, execute=True, device_capacity=cap, host_capacity=4 * 2 * rows * cols * 4)
    devs = ctx.devices
    dist = lambda: ctx.dist.stencil([rows, cols], [chunk_rows, cols], [1, 0], devs)  # noqa: E731
    a = ctx.create_array([rows, cols], "f32", dist(), 0)
    b = ctx.create_array([rows, cols], "f32", dist(), 0)
    work = ctx.dist.block_work([rows, cols], [16, 16], [chunk_rows, cols], devs)
    ctx.launch("ramp2d_f32", [rows, cols], [16, 16], work, [rows, cols, 1000, 0.0, 1.0, Arr(a)], "global [i, j] => write out[i,j]")
    ctx.synchronize()

    def run(n):
        nonlocal a, b
        for _ in range(n):
            ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, ALPHA, Arr(b), Arr(a)], ANN)
            ctx.flush()
            a, b = b, a
        ctx.synchronize()

    run(1)
    t0 = time.perf_counter()
    run(iters)
    dt = time.perf_counter() - t0
    try:
        rep = _json.loads(ctx.report_json())
        evictions = sum(int(w.get("evictions", 0)) for w in rep.get("workers", []))
    except Exception:  # noqa: BLE001
        evictions = None
    ctx.close()
    return {"value": rows * cols * iters / dt, "unit": "cell-updates/s", "cores": dv, "kind": "reference",
            "sample": f"heat2d {rows}x{cols} f32 x2 arrays, {chunk_rows}-row chunks over {dv} devices, device capacity "
                      f"{cap} B = 1/4 of each device's working set (acceptance c4), 1 warm-up + {iters} timed launches ({dt:.1f} s)",
            "evictions": evictions, "host": host_cpu()}


def run_contraction(ctx, n, steps, warmup, kind="bf16"):
    """BASELINE config C3 on one GPU: C (f32) = A x Bt^T, n^3, through the planner (one
    superblock per GPU) and the tcgen05 kernel; TFLOP/s from device events. kind "bf16": bf16
    operands (kind::f16); "tf32": f32 operands multiplied as TF32 (kind::tf32), C3's fp32 form."""
    from paper_2202_05549_b200 import Arr
    dev = ctx.devices
    kernel = f"matmul_nt_{kind}"
    et = "bf16" if kind == "bf16" else "f32"
    A = ctx.create_array([n, n], et, ctx.dist.single([n, n], dev[0]), 0)
    B = ctx.create_array([n, n], et, ctx.dist.single([n, n], dev[0]), 0)
    Cm = ctx.create_array([n, n], "f32", ctx.dist.single([n, n], dev[0]), 0)
    w = ctx.dist.block_work([n, n], [16, 16], [n, n], dev)
    ctx.launch(f"ramp2d_{et}", [n, n], [16, 16], w, [n, n, 1000, 0.0, 1.0, Arr(A)], "global [i, j] => write out[i,j]")
    ctx.launch(f"ramp2d_{et}", [n, n], [16, 16], w, [n, n, 997, 0.0, 1.0, Arr(B)], "global [i, j] => write out[i,j]")
    ann = "global [i, j] => write C[i,j], read A[i,:], read Bt[j,:]"

    def step():
        ctx.launch(kernel, [n, n], [16, 16], w, [n, n, n, Arr(Cm), Arr(A), Arr(B)], ann)
        ctx.flush()

    for _ in range(warmup):
        step()
    ctx.synchronize()
    k0, ms0 = ctx.kernel_time(kernel)
    ctx.profile_kernels(True)
    ctx.mark(0)
    for _ in range(steps):
        step()
    ctx.mark(1)
    elapsed = ctx.elapsed_ms()
    ctx.synchronize()
    ctx.profile_kernels(False)
    k1, ms1 = ctx.kernel_time(kernel)
    err = full_check(ctx, Cm, n, kind)
    for a in (A, B, Cm):
        ctx.delete_array(a)
    ctx.synchronize()
    flop = 2.0 * n ** 3
    kern_ms = (ms1 - ms0) / max(1, k1 - k0)
    return {"workload": f"{kernel} {n}^3 (C f32 = A {kind} x Bt^T {kind}), 1 superblock", "value": flop * steps / (elapsed / 1e3) / 1e12,
            "unit": "TFLOP/s", "steps": steps, "ms_per_step": elapsed / steps, "kernel_ms": kern_ms, "check": err}


def full_check(ctx, Cm, n, kind):
    """every element of C against an fp64 product (cuBLAS DGEMM, torch) of the same inputs,
    generated on the device from the ramp formula (bf16: rounded to nearest-even bf16, as the
    ramp2d_bf16 kernel stores them; tf32: the f32 values). Returns the max and mean relative
    error (the mean exposes a systematic bias) over all n^2 elements."""
    import torch
    dev = torch.device("cuda")

    def ramp(mod, off):
        i = torch.arange(n, dtype=torch.int64, device=dev)
        v = ((i[:, None] * 31 + i[None, :] * 17 + off) % mod).to(torch.float64) / mod
        v = v.to(torch.float32)
        if kind == "bf16":
            v = v.to(torch.bfloat16)
        return v.to(torch.float64)

    try:
        a = ramp(1000, 7)
        b = ramp(997, 7)
        want = a @ b.T
        del a, b
        got = torch.from_numpy(ctx.read(Cm)).to(dev)
        rel = (got.to(torch.float64) - want) / want.abs().clamp_min(1e-30)
        out = {"elements": n * n, "max_rel_err_vs_fp64": float(rel.abs().max()), "mean_rel_err_vs_fp64": float(rel.mean()),
               "reference": "fp64 cuBLAS product of the same inputs on the device"}
        del got, want, rel
    except Exception as e:  # noqa: BLE001
        out = {"unavailable": str(e)}
    torch.cuda.empty_cache()
    return out


def cublas_same_size(n, steps, warmup=2):
    """cuBLAS (torch.matmul, bf16 x bf16 -> bf16, its standard output type; ours writes f32, twice
    the output bytes) at the contraction's own size, timed like the contraction leg (warm-up
    launches, then `steps` back to back between two CUDA events), right after it so both run in
    the same power / clock state"""
    import torch
    a = torch.rand(n, n, device="cuda").to(torch.bfloat16)
    bt = torch.rand(n, n, device="cuda").to(torch.bfloat16)
    c = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    try:
        for _ in range(warmup):
            torch.matmul(a, bt.t(), out=c)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            torch.matmul(a, bt.t(), out=c)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / steps
    finally:
        del a, bt, c
        torch.cuda.empty_cache()
    return {"value": 2.0 * n ** 3 / (ms / 1e3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms, "steps": steps,
            "note": "torch.matmul bf16 x bf16^T -> bf16 (cuBLAS), same n, measured right after the tcgen05 leg"}


def cublas_tf32_peak(n=8192, reps=10):
    """measured dense TF32 peak of this box: torch.matmul on f32 with TF32 allowed (cuBLAS),
    best of `reps` back-to-back launches timed with CUDA events"""
    import torch
    a = torch.rand(n, n, device="cuda")
    b = torch.rand(n, n, device="cuda")
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        for _ in range(3):
            torch.matmul(a, b)
        best = 0.0
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            e1.synchronize()
            best = max(best, 2.0 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old
    del a, b
    torch.cuda.empty_cache()
    return best


def _timed(ctx, kernel, fn, steps):
    fn()
    ctx.synchronize()
    ctx.profile_kernels(True)
    k0, m0 = ctx.kernel_time(kernel)
    ctx.mark(0)
    for _ in range(steps):
        fn()
    ctx.mark(1)
    ms = ctx.elapsed_ms()
    ctx.synchronize()
    ctx.profile_kernels(False)
    k1, m1 = ctx.kernel_time(kernel)
    return ms / steps, (m1 - m0) / max(1, k1 - k0)


def ffma_probe(achieved):
    """the measured register-operand FFMA ceiling of this box (scripts/microbench/fma_dot.cu:
    16-term dot products, the assign kernel's inner-loop shape, best of 4 / 8 chains per thread)
    and the assign kernel's fraction of it"""
    import ctypes
    path = os.path.join(ROOT, "scripts", "microbench", "libfma_probe.so")
    try:
        lib = ctypes.CDLL(path)
        lib.mt_probe_ffma_dot.restype = ctypes.c_double
        lib.mt_probe_ffma_dot.argtypes = [ctypes.c_int]
        tmacs = lib.mt_probe_ffma_dot(20)
        if tmacs <= 0:
            raise RuntimeError("probe failed")
    except Exception as e:  # noqa: BLE001
        return {"measured_ffma_ceiling": {"unavailable": str(e)}}
    return {"measured_ffma_ceiling": {"value": tmacs * 1e12, "unit": "FFMA/s", "source": "scripts/microbench/fma_dot.cu (live, this run)"},
            "frac_of_measured_ffma": achieved / (tmacs * 1e12)}


def run_c4(ctx, hist_n, km_n, steps, hbm, cpu):
    """BASELINE config C4 on one GPU through the planner: histogram (reduce(+) into i64 bins)
    and int32 k-means (d=16, k=256). Step times from device events (all streams joined)."""
    from paper_2202_05549_b200 import Arr
    dev = ctx.devices
    out = {"histogram": [], "kmeans": None}
    n = hist_n
    for bins in (256, 65536):
        x = ctx.create_array([n], "i32", ctx.dist.single([n], dev[0]), 0)
        h = ctx.create_array([bins], "i64", ctx.dist.single([bins], dev[0]), 0)
        w = ctx.dist.block_work([n], [256], [n], dev)
        ctx.launch("hpattern1d", [n], [256], w, [n, bins, 12345, Arr(x)], "global i => write out[i]")

        def step():
            ctx.launch("histogram", [n], [256], w, [n, bins, Arr(x), Arr(h)], "global i => read x[i], reduce(+) hist[:]")
            ctx.flush()

        ms, _ = _timed(ctx, "histogram", step, steps)
        ok = int(ctx.read(h).sum()) == n
        gbs = 4.0 * n / (ms / 1e3) / 1e9
        out["histogram"].append({"workload": f"histogram n={n} i32 -> {bins} i64 bins", "value": n / (ms / 1e3), "unit": "elements/s", "ms_per_step": ms,
                                 "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                                              "note": "4 B/element; step time (plan + partial + reduce tree + copy-back) over device events"},
                                 "total_count_check": ok})
        ctx.delete_array(x)
        ctx.delete_array(h)
        ctx.synchronize()
    n, k, d = km_n, 256, 16
    pts = ctx.create_array([n, d], "i32", ctx.dist.single([n, d], dev[0]), 0)
    asg = ctx.create_array([n], "i32", ctx.dist.single([n], dev[0]), 0)
    cen = ctx.create_array([k, d], "i32", ctx.dist.single([k, d], dev[0]), 0)
    sums = ctx.create_array([k, d], "i64", ctx.dist.single([k, d], dev[0]), 0)
    cnts = ctx.create_array([k], "i64", ctx.dist.single([k], dev[0]), 0)
    ctx.launch("ipattern2d_i32", [n, d], [256, 16], ctx.dist.block_work([n, d], [256, 16], [n, d], dev), [n, d, 1000, Arr(pts)],
               "global [i, j] => write out[i,j]")
    wk = ctx.dist.block_work([k, d], [16, 16], [k, d], dev)
    ctx.launch("ipattern2d_i32", [k, d], [16, 16], wk, [k, d, 997, Arr(cen)], "global [i, j] => write out[i,j]")
    w1 = ctx.dist.block_work([n], [256], [n], dev)

    def assign():
        ctx.launch("kmeans_assign_i32", [n], [256], w1, [n, k, d, Arr(asg), Arr(pts), Arr(cen)],
                   "global i => write assign[i], read points[i,:], read centroids[:,:]")
        ctx.flush()

    def update():
        ctx.launch("kmeans_update_i32", [n], [256], w1, [n, d, Arr(pts), Arr(asg), Arr(sums), Arr(cnts)],
                   "global i => read points[i,:], read assign[i], reduce(+) sums[:,:], reduce(+) counts[:]")
        ctx.flush()

    a_ms, a_kms = _timed(ctx, "kmeans_assign_i32", assign, 2)
    u_ms, u_kms = _timed(ctx, "kmeans_update_i32", update, steps)
    ok = int(ctx.read(cnts).sum()) == n  # reduce(+) overwrites its destination each launch (planner.cpp:507-509)
    for a in (pts, asg, cen, sums, cnts):
        ctx.delete_array(a)
    ctx.synchronize()
    triples = float(n) * k * d
    fma_peak = 148 * 128 * 1.965e9  # nominal FP32 FFMA per clk per SM x SMs x max clock
    ubytes = n * (d + 1) * 4
    out["kmeans"] = {"workload": f"int32 k-means n={n} d={d} k={k}", "value": n / ((a_ms + u_ms) / 1e3), "unit": "points/s (assign + update)",
                     "assign": {"ms": a_kms, "roofline": {"bound": "fp32 fma pipe", "achieved": triples / (a_kms / 1e3), "peak": fma_peak,
                                                           "unit": "(point, centroid, dim) terms/s", "frac": triples / (a_kms / 1e3) / fma_peak,
                                                           "peak_kind": "derived: 148 SM x 128 FFMA/clk x 1.965 GHz (nominal; a three-register FFMA "
                                                                        "issues every 2nd cycle per SMSP, see measured_ffma_ceiling); one exact "
                                                                        "FFMA per term, the u32 / int64 tiers take over beyond 2^24",
                                                           "frac_of_imad_bound": triples / (a_kms / 1e3) / (148 * 64 * 1.965e9),
                                                           **ffma_probe(triples / (a_kms / 1e3))}},
                     "update": {"ms": u_ms, "kernel_ms": u_kms, "roofline": {"bound": "hbm", "achieved": ubytes / (u_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                                                           "frac": ubytes / (u_ms / 1e3) / 1e9 / hbm,
                                                           "note": "68 B/point read-only stream over the step time (consecutive updates overlap)"}},
                     "count_check": ok}
    if cpu:
        import oracle
        try:
            out["cpu_baseline"] = cpu_c4(oracle)
        except Exception as e:  # noqa: BLE001
            out["cpu_baseline"] = {"unavailable": str(e)}
    return out


def cpu_c4(oracle):
    """reference CPU executor (oracle/_ref) on bounded samples of the C4 workloads"""
    from paper_2202_05549_b200 import Arr
    threads = oracle.reference().host_threads()
    dv = max(1, min(threads, 64))
    res = {}
    n, bins = 1_000_000_000, 256
    # a 1e9-element sample puts 250 MB chunks on each of 16 devices: above the reference's
    # default staging threshold (64 MiB, memory.hpp:50) and device capacity (256 MiB), so both
    # are raised (the workload is in-core on the CPU; the limits only model a device)
    big = {"staging_threshold": 1 << 40, "device_capacity": 1 << 40}
    ctx = oracle.reference_context(workers=1, devices=dv, execute=True, **big)
    devs = ctx.devices
    per = (n + dv - 1) // dv
    per = (per + 255) // 256 * 256
    x = ctx.create_array([n], "i32", ctx.dist.row([n], per, devs), 0)
    h = ctx.create_array([bins], "i64", ctx.dist.replicated([bins], devs), 0)
    w = ctx.dist.block_work([n], [256], [per], devs)
    ctx.launch("hpattern1d", [n], [256], w, [n, bins, 12345, Arr(x)], "global i => write out[i]")
    ctx.synchronize()
    t0 = time.perf_counter()
    ctx.launch("histogram", [n], [256], w, [n, bins, Arr(x), Arr(h)], "global i => read x[i], reduce(+) hist[:]")
    ctx.synchronize()
    dt = time.perf_counter() - t0
    ctx.close()
    res["histogram"] = {"value": n / dt, "unit": "elements/s", "cores": dv, "kind": "reference", "sample": f"n={n}, {bins} bins, {dt:.1f} s"}
    n, k, d = 1_000_000, 256, 16  # 1e6 points
    ctx = oracle.reference_context(workers=1, devices=dv, execute=True, **big)
    devs = ctx.devices
    per = ((n + dv - 1) // dv + 255) // 256 * 256
    pts = ctx.create_array([n, d], "i32", ctx.dist.row([n, d], per, devs), 0)
    asg = ctx.create_array([n], "i32", ctx.dist.row([n], per, devs), 0)
    cen = ctx.create_array([k, d], "i32", ctx.dist.replicated([k, d], devs), 0)
    sums = ctx.create_array([k, d], "i64", ctx.dist.replicated([k, d], devs), 0)
    cnts = ctx.create_array([k], "i64", ctx.dist.replicated([k], devs), 0)
    ctx.launch("ipattern2d_i32", [n, d], [256, 16], ctx.dist.block_work([n, d], [256, 16], [per, d], devs), [n, d, 1000, Arr(pts)],
               "global [i, j] => write out[i,j]")
    ctx.launch("ipattern2d_i32", [k, d], [16, 16], ctx.dist.block_work([k, d], [16, 16], [k, d], devs), [k, d, 997, Arr(cen)],
               "global [i, j] => write out[i,j]")
    ctx.synchronize()
    w1 = ctx.dist.block_work([n], [256], [per], devs)
    t0 = time.perf_counter()
    ctx.launch("kmeans_assign_i32", [n], [256], w1, [n, k, d, Arr(asg), Arr(pts), Arr(cen)],
               "global i => write assign[i], read points[i,:], read centroids[:,:]")
    ctx.launch("kmeans_update_i32", [n], [256], w1, [n, d, Arr(pts), Arr(asg), Arr(sums), Arr(cnts)],
               "global i => read points[i,:], read assign[i], reduce(+) sums[:,:], reduce(+) counts[:]")
    ctx.synchronize()
    dt = time.perf_counter() - t0
    ctx.close()
    res["kmeans"] = {"value": n / dt, "unit": "points/s (assign + update)", "cores": dv, "kind": "reference", "sample": f"n={n}, k={k}, d={d}, {dt:.1f} s"}
    return res


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    try:
        import oracle
        threads = oracle.reference().host_threads() if hasattr(oracle.reference(), "host_threads") else (os.cpu_count() or 1)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"impl": "reference", "unavailable": f"reference CPU executor not loadable: {e}"}))
        return
    devices = max(1, min(threads, 64))
    rows = sample_rows(args.cpu_rows, devices)
    cols = args.cols
    # the shared protocol (CPU_ROWS band, warm-up launches in the same context), each step one
    # heat iteration over the band; the step count is capped so the arm ends within minutes
    steps = max(1, min(args.steps, 60))
    # the CPU warm-up is the protocol's own (first-touch of the band), not the GPU's W
    rate, dt = cpu_reference_rate(rows, cols, steps, devices, warmup=CPU_WARMUP, bounds_check=args.cpu_bounds_check == "on")
    sample = (f"{rows}x{cols} band of the {args.rows}x{args.cols} grid, {devices} chunks (stencil_dist halo [1,0]), 1 worker x {devices} "
              f"device threads, {CPU_WARMUP} warm-up + {steps} timed launches"
              + ("" if args.cpu_bounds_check == "on" else ", array_view bounds checks off"))
    print(json.dumps({
        "metric": METRIC, "impl": "reference", "value": rate, "unit": "cell-updates/s", "n_gpus": args.gpus, "steps": steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3 / steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (ramp2d_f32 pattern)",
        "config": {"workload": "heat2d 2D 5-point stencil f32, row-block stencil distribution", "rows": rows, "cols": cols, "iterations_per_step": 1},
        "cpu_baseline": {"value": rate, "unit": "cell-updates/s", "cores": devices, "kind": "reference", "sample": sample, "host": host_cpu()},
        "e2e": {"value": rate, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# FP64-pipe instructions per pair interaction of nbody_tiled_k<3, 8>: DADD 9 + DMUL 10 + DFMA 10
# (the two MUFU seeds run on the XU pipe); ncu sm__sass_thread_inst_executed_op_{dadd,dmul,dfma}
# in the ratio 9:10:10, profiles/round2/ncu/nbody_summary.txt
NBODY_DP_PER_PAIR = 29


def run_nbody(n, steps, cpu):
    """nbody_like (the reference kernel, kernels.cpp:369-401: all pairs, f64, bit-exact) on one
    GPU through the planner: pair interactions per second, roofline = FP64-pipe instructions
    (NBODY_DP_PER_PAIR per pair) against 148 SMs x 64 FP64 lanes x the SM clock; the reference
    CPU executor on an n=8192 sample beside it"""
    import numpy as np

    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    d = 3
    with mb.context(workers=1, devices=1, num_gpus=1) as ctx:
        dv = ctx.devices
        pos = ctx.create_array([n, d], "f64", ctx.dist.single([n, d], dv[0]), 0)
        force = ctx.create_array([n, d], "f64", ctx.dist.single([n, d], dv[0]), 0)
        ctx.write(pos, np.random.default_rng(1).standard_normal((n, d)))
        w = ctx.dist.block_work([n], [256], [n], dv)

        def step():
            ctx.launch("nbody_like", [n], [256], w, [n, d, Arr(force), Arr(pos)], "global i => write force[i,:], read pos[:,:]")
            ctx.flush()

        ms, kms = _timed(ctx, "nbody_like", step, steps)
    pairs = float(n) * (n - 1)
    dp_peak = 148 * 64 * 1.965e9
    out = {"workload": f"nbody_like n={n} d={d} f64 all pairs", "value": pairs / (ms / 1e3), "unit": "pair interactions/s", "ms_per_step": ms,
           "roofline": {"bound": "fp64 pipe", "achieved": pairs * NBODY_DP_PER_PAIR / (kms / 1e3), "peak": dp_peak, "unit": "FP64 instructions/s",
                        "frac": pairs * NBODY_DP_PER_PAIR / (kms / 1e3) / dp_peak,
                        "peak_kind": "derived: 148 SM x 64 FP64 lanes x 1.965 GHz (B200 FP64 37 TFLOP/s = 2 x that)",
                        "note": f"{NBODY_DP_PER_PAIR} FP64-pipe instructions per pair (IEEE-rounded sqrt and divide for bit-exactness)"}}
    if cpu:
        try:
            import oracle
            threads = oracle.reference().host_threads()
            dvn = max(1, min(threads, 64))
            m = 8192
            rctx = oracle.reference_context(workers=1, devices=dvn, execute=True)
            devs = rctx.devices
            per = ((m + dvn - 1) // dvn + 15) // 16 * 16
            p2 = rctx.create_array([m, d], "f64", rctx.dist.replicated([m, d], devs), 0)
            f2 = rctx.create_array([m, d], "f64", rctx.dist.row([m, d], per, devs), 0)
            rctx.launch("ramp2d", [m, d], [16, 1], rctx.dist.block_work([m, d], [16, 1], [m, d], devs[:1]), [m, d, 1000, -0.5, 1e-3, Arr(p2)],
                        "global [i, j] => write out[i,j]")
            rctx.synchronize()
            t0 = time.perf_counter()
            rctx.launch("nbody_like", [m], [16], rctx.dist.block_work([m], [16], [per], devs), [m, d, Arr(f2), Arr(p2)],
                        "global i => write force[i,:], read pos[:,:]")
            rctx.synchronize()
            dt = time.perf_counter() - t0
            rctx.close()
            out["cpu_baseline"] = {"value": float(m) * (m - 1) / dt, "unit": "pair interactions/s", "cores": dvn, "kind": "reference",
                                   "sample": f"n={m}, d={d}, 1 worker x {dvn} device threads ({dt:.1f} s)"}
        except Exception as e:  # noqa: BLE001
            out["cpu_baseline"] = {"unavailable": str(e)}
    return out


def link_bandwidth(gib=4):
    """pinned host <-> HBM copy bandwidth (GB/s): H2D, D2H and each way with both at once"""
    import torch
    n = gib << 30
    h_src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d_src = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name, fn in [("h2d", lambda: d_dst.copy_(h_src, non_blocking=True)), ("d2h", lambda: h_dst.copy_(d_src, non_blocking=True))]:
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        res[name] = 3 * n / (time.perf_counter() - t0) / 1e9
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        with torch.cuda.stream(s1):
            d_dst.copy_(h_src, non_blocking=True)
        with torch.cuda.stream(s2):
            h_dst.copy_(d_src, non_blocking=True)
    torch.cuda.synchronize()
    res["duplex_each_way"] = 3 * n / (time.perf_counter() - t0) / 1e9
    del h_src, h_dst, d_src, d_dst
    torch.cuda.empty_cache()
    return res


def run_ooc(rows, cols, chunk_rows, capacity_gib, host_gib, iters, warmup, lookahead=0):
    """BASELINE config C5 (out-of-core heat2d) on one GPU with the pinned-host spill tier: two
    rows x cols f32 arrays in chunk_rows-row chunks (halo [1,0]) with the device capacity capped.
    Each iteration reads one array and overwrites the other (dead, never restored), so the
    minimum traffic is the part of one array that does not fit, each way; the bound is that
    volume over the measured duplex pinned bandwidth. Device-event timing."""
    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    bw = link_bandwidth()
    cr = chunk_rows
    cap = int(capacity_gib * (1 << 30))
    la = lookahead or 3 * (rows // cr) * 3
    ctx = mb.context(workers=1, devices=1, num_gpus=1, device_capacity=cap, host_capacity=int(host_gib * (1 << 30)), lookahead_tasks=la,
                     retain_plan=False)
    devs = ctx.devices
    dist = lambda: ctx.dist.stencil([rows, cols], [cr, cols], [1, 0], devs)  # noqa: E731
    a = ctx.create_array([rows, cols], "f32", dist(), 0)
    b = ctx.create_array([rows, cols], "f32", dist(), 0)
    work = ctx.dist.block_work([rows, cols], [16, 16], [cr, cols], devs)
    ctx.launch("ramp2d_f32", [rows, cols], [16, 16], work, [rows, cols, 1000, 0.0, 1.0, Arr(a)], "global [i, j] => write out[i,j]")
    t_setup = time.perf_counter()
    for _ in range(warmup):
        ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, ALPHA, Arr(b), Arr(a)], ANN)
        ctx.flush()
        a, b = b, a
    ctx.synchronize()
    t_setup = time.perf_counter() - t_setup
    s0 = ctx.exec_stats()
    ctx.mark(0)
    for _ in range(iters):
        ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, ALPHA, Arr(b), Arr(a)], ANN)
        ctx.flush()
        a, b = b, a
    ctx.mark(1)
    ms = ctx.elapsed_ms()
    ctx.synchronize()
    s1 = ctx.exec_stats()
    ctx.close()
    wset = 2 * rows * cols * 4
    h2d = (s1["spill_bytes_h2d"] - s0["spill_bytes_h2d"]) / iters
    d2h = (s1["spill_bytes_d2h"] - s0["spill_bytes_d2h"]) / iters
    minimum = max(0, wset // 2 - cap)
    survey_bound = max(0, wset - cap)  # SURVEY 8d's looser (working set - resident) each way
    per_iter = ms / iters / 1e3
    bound = minimum / (bw["duplex_each_way"] * 1e9)
    return {"workload": f"out-of-core heat2d {rows}x{cols} f32 x2 arrays, {cr}-row chunks, device capacity {capacity_gib} GiB",
            "working_set_gib": wset / 2**30, "capacity_gib": capacity_gib, "iters": iters, "s_per_iter": per_iter,
            "value": rows * cols / per_iter, "unit": "cell-updates/s", "h2d_gib_per_iter": h2d / 2**30, "d2h_gib_per_iter": d2h / 2**30,
            "min_gib_each_way_per_iter": minimum / 2**30, "moved_over_min": max(h2d, d2h) / minimum if minimum else None,
            "survey_bound_gib_each_way": survey_bound / 2**30,
            "time_over_survey_bound": per_iter / (survey_bound / (bw["duplex_each_way"] * 1e9)) if survey_bound else None,
            "link_gbs": bw, "bound_s_per_iter": bound, "time_over_bound": per_iter / bound if bound else None,
            "lookahead_tasks": la, "warmup_s": t_setup, "evictions": s1["evictions"] - s0["evictions"],
            "scale_note": "BASELINE configs[4] asks for a 400 GB array; this box has one B200 (180 GB HBM) and ~196 GB of host RAM, "
                          "so the pinned host tier cannot hold the ~250 GB that must live off-device: the leg runs a working set larger "
                          "than the capped device capacity instead (profiles/round1/ooc_192gib_over_hbm.json: 192 GiB on the full HBM)"}


# launches per mt_flush in the C1 leg: a 10-launch submission is replayed as one CUDA graph whose
# edges run across iterations (profiles/round1/c1_flush_sweep.md)
C1_PER_FLUSH = 10


def same_size_copy_gbs(nbytes, iters=200):
    """a plain device copy of one array of the C1 grid (torch copy_, back to back, CUDA events):
    what the copy peak's 1 GiB figure becomes at this size (the read and written 64 MiB sit in
    and around the L2), the line the C1 step is compared with beside the HBM peak"""
    import torch
    a = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda").uniform_()
    b = torch.empty_like(a)
    for _ in range(20):
        b.copy_(a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    del a, b
    torch.cuda.empty_cache()
    return {"achieved": 2 * nbytes / (us / 1e6) / 1e9, "unit": "GB/s", "us_per_copy": us,
            "what": f"torch copy_ of {nbytes >> 20} MiB device to device, {iters} back to back"}


def run_c1(iters, ref_iters, hbm, cpu, strip=0, chunks=4):
    """BASELINE configs[0] (the reference's CPU scenario): heat2d 4096^2 f32, row-block stencil
    distribution into 4 chunks, one distributed launch per iteration, on one GPU (4 logical
    devices), next to the reference CPU executor on the same grid and chunking."""
    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr
    rows = cols = 4096
    with mb.context(workers=1, devices=chunks, num_gpus=1, retain_plan=False) as ctx:
        a, b, work = setup_heat(ctx, rows, cols, chunks, strip=strip)

        def run(n):
            # the reference's repeat/swap loop in one native call (mt_launch_repeat); repeated
            # launches replay their memoized plan (planner plan cache)
            nonlocal a, b
            ctx.launch_repeat("heat2d", [rows, cols], [16, 16], work, [rows, cols, ALPHA, Arr(b), Arr(a)], ANN, n, swap=(a, b),
                              flush_every=C1_PER_FLUSH)
            ctx.flush()
            if n % 2:
                a, b = b, a

        run(3 * C1_PER_FLUSH)
        ctx.synchronize()
        ctx.mark(0)
        run(iters)
        ctx.mark(1)
        ms = ctx.elapsed_ms() / iters
        ctx.synchronize()
        st = ctx.exec_stats()
        hits = ctx.plan_cache_hits()
    gbs = BYTES_PER_CELL * rows * cols / (ms / 1e3) / 1e9
    same = same_size_copy_gbs(rows * cols * 4)
    out = {"workload": f"heat2d {rows}x{cols} f32, 4 chunks (stencil_dist halo [1,0]), {iters} iterations, one launch per iteration "
                       f"(mt_launch_repeat with the a/b swap), handed to the executor every {C1_PER_FLUSH} launches"
                       + (f"; 3 superblocks per chunk ({strip}-row halo-facing strips, interior)" if strip else ""),
           "value": rows * cols / (ms / 1e3), "unit": "cell-updates/s", "ms_per_iter": ms,
           "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                        "note": "step time incl. planning, halo copies and graph launch; the 64 MiB grid is kept L2-resident between steps (outputs stored with the default policy, dead inputs read evict-first), so the HBM figure is a reference line, not a ceiling",
                        "same_size_copy": same, "frac_of_same_size_copy": gbs / same["achieved"] if same else None},
           "graph_replays": st.get("graph_replays"), "plan_cache_hits": hits, "fused_halo_copies": st.get("fused_copies"),
           "halo_copies": st.get("copies")}
    if cpu:
        try:
            rate, dt = cpu_reference_rate(rows, cols, ref_iters, 4, warmup=1)
            out["cpu_baseline"] = {"value": rate, "unit": "cell-updates/s", "cores": 4, "kind": "reference",
                                   "sample": f"the same 4096^2 grid and 4 chunks (one device thread each), 1 warm-up + {ref_iters} timed iterations ({dt:.1f} s)"}
        except Exception as e:  # noqa: BLE001
            out["cpu_baseline"] = {"unavailable": str(e)}
    return out


def run_b200(args):
    import numpy as np
    import torch

    import paper_2202_05549_b200 as mb
    from paper_2202_05549_b200 import Arr

    ws, rank, local = dist_env()
    rows, cols = args.rows, args.cols
    if ws > 1:
        # one process per GPU: worker `rank` of a ws-worker system; every rank plans the whole
        # (identical) plan and executes its own worker's tasks; halo rows move through the
        # GPU-driven IPC rings (executor.cu, inter-process send/recv)
        import torch.distributed as dist
        gpu = local % torch.cuda.device_count()
        torch.cuda.set_device(gpu)
        # NCCL for the timing reductions when every rank has its own GPU; gloo when ranks share one
        # (functional test of the multi-process path on a single-GPU box)
        dist.init_process_group("nccl" if torch.cuda.device_count() >= ws else "gloo")
        gloo = dist.new_group(backend="gloo")
        ctx = mb.context(workers=ws, devices=1, worker_rank=rank, gpu_base=gpu, retain_plan=False)
        ctx.connect_peers(gloo)
        args.matmul_n, args.c4 = 0, False  # the C3/C4 legs are single-GPU workloads: reported at N=1 only
    else:
        ctx = mb.context(workers=1, devices=1, num_gpus=1, retain_plan=False)
    a, b, work = setup_heat(ctx, rows, cols, ws, strip=args.strip if ws > 1 else 0)
    ctx.synchronize()

    def step():
        nonlocal a, b
        ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, ALPHA, Arr(b), Arr(a)], ANN)
        ctx.flush()
        a, b = b, a

    for _ in range(args.warmup):
        step()
    ctx.synchronize()
    stats0 = ctx.exec_stats()
    ctx.profile_kernels(True)
    k0, ms0 = ctx.kernel_time("heat2d")
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    ctx.mark(0)
    for _ in range(args.steps):
        step()
    ctx.mark(1)
    elapsed = ctx.elapsed_ms()
    ctx.synchronize()
    clocks = sampler.stop()
    ctx.profile_kernels(False)
    k1, ms1 = ctx.kernel_time("heat2d")
    stats1 = ctx.exec_stats()
    elapsed = barrier_max(elapsed, ws)
    cells = rows * cols * args.steps  # strong scaling: the whole grid, split over the ranks
    value = cells / (elapsed / 1e3)
    # heat2d kernel time per step on this rank (its superblocks run back to back or overlapped)
    kern_ms = (ms1 - ms0) / max(1, args.steps)
    achieved = BYTES_PER_CELL * (rows // ws) * cols / (kern_ms / 1e3) / 1e9
    peak, peak_kind = peaks()

    # best and median of 5 further timed runs (K/5 steps each, device events, max
    # over ranks) next to the K-step figure
    repeats = []
    for _ in range(5):
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()
        ctx.mark(0)
        for _ in range(max(1, args.steps // 5)):
            step()
        ctx.mark(1)
        repeats.append(rows * cols * max(1, args.steps // 5) / (barrier_max(ctx.elapsed_ms(), ws) / 1e3))
    ctx.synchronize()
    runs = {"best": max(repeats), "median": statistics.median(repeats), "runs": len(repeats), "steps_per_run": max(1, args.steps // 5)}

    # e2e through the public API with host buffers
    e2e = None
    if args.e2e_runs > 0:
        # host buffers: the whole grid at N=1; at N>1 each rank holds only its chunk's box
        # (rows of its block plus halo rows) and moves it with mt_array_{write,read}_box_async,
        # so the job as a whole uploads and downloads the grid once per step
        box = None
        if ws > 1:
            mine = [c for c in ctx.chunks(a) if c.home[0] == rank][0]
            box = (mine.lo, mine.hi)
        hshape = (rows, cols) if box is None else (box[1][0] - box[0][0], cols)
        host_in = (torch.empty if box is None else torch.zeros)(hshape, dtype=torch.float32, pin_memory=True)
        host_out = [torch.empty(hshape, dtype=torch.float32, pin_memory=True) for _ in range(2)]
        hin = host_in.numpy()
        hout = host_out[0].numpy()
        if box is None:
            ctx.lib.check(ctx.lib.array_read(ctx.h, a, hin.ctypes.data, hin.nbytes))
        else:
            ctx.read_async(a, host_in, box=box)
            ctx.synchronize()
        # whole job per step: every chunk is uploaded whole (halo rows included), every cell is
        # downloaded once (from the lowest-id chunk holding it)
        h2d_bytes = 4 * sum((c.hi[0] - c.lo[0]) * (c.hi[1] - c.lo[1]) for c in ctx.chunks(a)) if box else rows * cols * 4
        d2h_bytes = rows * cols * 4

        def sync_barrier():
            ctx.synchronize()
            if ws > 1:
                import torch.distributed as dist
                dist.barrier()

        # (1) sequential: each step uploads the grid, iterates, reads the grid back, synchronously
        times = []
        for run in range(args.e2e_runs + 1):
            sync_barrier()
            t0 = time.perf_counter()
            if box is None:
                ctx.lib.check(ctx.lib.array_write(ctx.h, a, hin.ctypes.data, hin.nbytes))
            else:
                ctx.write_async(a, host_in, box=box)
            for _ in range(args.e2e_iters):
                step()
            if box is None:
                ctx.lib.check(ctx.lib.array_read(ctx.h, a, hout.ctypes.data, hout.nbytes))
            else:
                ctx.read_async(a, host_out[0], box=box)
                ctx.synchronize()
            dt = barrier_max(time.perf_counter() - t0, ws)
            if run > 0:  # first run is warm-up
                times.append(dt)
        seq = rows * cols * args.e2e_iters / (sum(times) / len(times))
        # (2) pipelined: the same steps queued back to back through mt_array_write_async /
        # mt_array_read_async on `e2e_sets` array sets (triple buffering by default), so step
        # s+1's upload (into a set nobody uses) and step s-1's download (from another) run in
        # both PCIe directions at once under step s's iterations; with two sets the upload
        # would wait for the download from the same set. Every step still moves its whole
        # input in and its whole result out inside the timed region
        pipe = None
        if args.e2e_pipeline > 0:
            nsets = max(2, args.e2e_sets)
            sets = [(a, b)] + [setup_heat(ctx, rows, cols, ws, strip=args.strip if ws > 1 else 0)[:2] for _ in range(nsets - 1)]

            def pstep(s):
                x, y = sets[s % nsets]
                ctx.write_async(x, host_in, box=box)
                for _ in range(args.e2e_iters):
                    ctx.launch("heat2d", [rows, cols], [16, 16], work, [rows, cols, ALPHA, Arr(y), Arr(x)], ANN)
                    x, y = y, x
                ctx.read_async(x, host_out[s % 2], box=box)
                ctx.flush()

            pstep(0)
            sync_barrier()
            t0 = time.perf_counter()
            for s in range(args.e2e_pipeline):
                pstep(s)
            ctx.synchronize()
            pdt = barrier_max(time.perf_counter() - t0, ws)
            pipe = rows * cols * args.e2e_iters * args.e2e_pipeline / pdt
            for st in sets[1:]:
                for arr in st:
                    ctx.delete_array(arr)
            ctx.synchronize()
        dt = max(times) if times else float("nan")
        e2e = {"value": pipe if pipe else seq, "unit": "cell-updates/s", "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes,
               "iterations_per_step": args.e2e_iters, "steps": args.e2e_pipeline if pipe else len(times),
               "note": ("step = upload the grid from pinned host memory + e2e iterations + read the grid back, through the public API"
                        + (" (each rank its own chunk box, mt_array_*_box_async)" if box else "") + "; "
                        + (f"steps pipelined with mt_array_write_async / mt_array_read_async over {max(2, args.e2e_sets)} array sets (uploads, "
                           "downloads and kernels overlap)" if pipe else "synchronous mt_array_write / mt_array_read")
                        + "; wall clock, max over ranks"),
               "sequential": {"value": seq, "steps": len(times), "worst_step_s": dt,
                              "note": "each step synchronous: upload, iterations, download"}}
        del host_in, host_out
        try:  # hand the pinned host buffers back (torch caches freed pinned blocks) before the C5 leg pins its own
            torch._C._host_emptyCache()
        except Exception:  # noqa: BLE001
            pass

    cpu = None
    if rank == 0 and ws == 1 and args.cpu_baseline:  # N=1 only (the reference arm covers N>1)
        try:
            cpu = cpu_heat_baseline(cols, rows, want_rows=args.cpu_rows, steps=args.cpu_iters)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "cell-updates/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    def leg(fn, *a, **kw):
        # a secondary leg that fails is reported as unavailable; the heat line above stands
        try:
            return fn(*a, **kw)
        except Exception as e:  # noqa: BLE001
            import traceback
            traceback.print_exc()
            return {"unavailable": f"{type(e).__name__}: {e}"}

    contraction = None
    if args.matmul_n > 0:
        contraction = leg(run_contraction, ctx, args.matmul_n, args.matmul_steps, 2)
    if contraction is not None and "unavailable" not in contraction:
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                pk = json.load(f)
            tpeak, tburst = float(pk["bf16_tflops_sustained"]), float(pk["bf16_tflops"])
        except Exception:
            tpeak, tburst = 1400.0, 1590.0
        kach = 2.0 * args.matmul_n ** 3 / (contraction["kernel_ms"] / 1e3) / 1e12
        # the timed region is a few 50 ms launches: a kernel timed alone, so the burst figure
        contraction["roofline"] = {"bound": "tensor", "achieved": kach, "peak": tburst, "unit": "TFLOP/s", "frac": kach / tburst,
                                   "peak_kind": "measured burst (cuBLAS bf16 8192^3, best of 10)", "frac_of_sustained": kach / tpeak,
                                   "kernel": "gemm_bf16_nt_2sm_kernel<bf16, wide> (CTA pairs, 256x512 tiles: two tcgen05.mma cta_group::2 M256 N256 per K step, TMA, TMEM, dynamic tile counter)"}
        try:
            cb = cublas_same_size(args.matmul_n, args.matmul_steps)
            contraction["cublas_same_size"] = cb
            contraction["roofline"]["frac_of_cublas_same_size"] = contraction["value"] / cb["value"]
        except Exception as e:  # noqa: BLE001
            contraction["cublas_same_size"] = {"unavailable": str(e)}
        t32 = leg(run_contraction, ctx, args.matmul_n, args.tf32_steps, 1, "tf32") if args.tf32_steps > 0 else None
        if t32 is not None and "unavailable" in t32:
            contraction["tf32"] = t32
        elif t32 is not None:
            k32 = 2.0 * args.matmul_n ** 3 / (t32["kernel_ms"] / 1e3) / 1e12
            try:
                p32, p32_kind = cublas_tf32_peak(), "measured here: cuBLAS TF32 (torch.matmul f32, allow_tf32) 8192^3, best of 10"
            except Exception as e:  # noqa: BLE001
                p32, p32_kind = tburst / 2, f"half the measured bf16 burst (cuBLAS TF32 measurement failed: {e})"
            t32["roofline"] = {"bound": "tensor", "achieved": k32, "peak": p32, "unit": "TFLOP/s", "frac": k32 / p32, "peak_kind": p32_kind,
                               "frac_of_half_bf16_burst": k32 / (tburst / 2),
                               "kernel": "tf32_rne rounding pass + gemm_bf16_nt_2sm_kernel<TF32, wide> (tcgen05.mma cta_group::2 kind::tf32 M256 N256 x2, TMA, TMEM); "
                                         "kernel_ms includes the rounding pass"}
            contraction["tf32"] = t32
        if rank == 0 and args.cpu_baseline:
            try:
                contraction["cpu_baseline"] = cpu_matmul_baseline()
            except Exception as e:  # noqa: BLE001
                contraction["cpu_baseline"] = {"unavailable": str(e)}
    nbody = None
    if ws == 1 and args.nbody_n > 0:
        nbody = leg(run_nbody, args.nbody_n, 3, rank == 0 and args.cpu_baseline)
    c1 = None
    if ws == 1 and args.c1:
        c1 = leg(run_c1, 100, args.c1_ref_iters, peaks()[0], rank == 0 and args.cpu_baseline, strip=args.c1_strip)
    c4 = None
    if args.c4:
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                hbm = float(json.load(f)["hbm_gbs"])
        except Exception:
            hbm = 6650.0
        c4 = leg(run_c4, ctx, args.hist_n, args.km_n, 5, hbm, rank == 0 and args.cpu_baseline)
    traffic = ncu_traffic("heat2d_tma_ncu_summary.json", rows // ws, cols)
    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "cell-updates/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (ramp2d_f32 pattern generated on device)",
            "config": {"workload": f"heat2d 2D 5-point stencil f32 {rows}x{cols} over {ws} GPU(s), row-block stencil distribution halo [1,0], "
                                   "one distributed launch per step (plan + halo exchange + kernel)",
                       "rows": rows, "cols": cols, "alpha": ALPHA, "parallelism": f"dp{ws} (row blocks, one process per GPU)",
                       "superblocks_per_gpu": 3 if ws > 1 else 1, "l2": "inputs (2 x 16 GiB total) >> L2, no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic[0] if traffic else None, "traffic_source": traffic[1] if traffic else None,
                         "kernel": "heat2d_tma_kernel (TMA-staged rows, mbarrier ring)", "kernel_ms": kern_ms, "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": BYTES_PER_CELL * (rows // ws) * cols},
            "clocks": clocks,
            "repeats": runs,
            "gpu_launches": int(stats1.get("kernels", 0) - stats0.get("kernels", 0)),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "contraction": contraction,
            "reductions": c4,
            "small_grid": c1,
            "nbody": nbody,
        }
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()  # no rank may unmap its mailbox while a peer still writes into it
    ctx.close()
    if ws == 1 and args.ooc_gib > 0:
        # C5: spill-tier heat2d with both arrays in 1 GiB chunks and one array larger than the
        # capped device capacity (a fresh context; the main one is closed)
        import torch
        torch.cuda.empty_cache()
        try:
            rows_ooc = int(args.ooc_gib * (1 << 30)) // (2 * 4 * cols) // 4096 * 4096
            out["out_of_core"] = run_ooc(rows_ooc, cols, 4096, args.ooc_cap_gib, max(8.0, args.ooc_gib - args.ooc_cap_gib + 8.0), args.ooc_iters, 2)
        except Exception as e:  # noqa: BLE001
            out["out_of_core"] = {"unavailable": str(e)}
        if args.cpu_baseline and "unavailable" not in out["out_of_core"]:
            try:
                out["out_of_core"]["cpu_baseline"] = cpu_ooc_baseline()
            except Exception as e:  # noqa: BLE001
                out["out_of_core"]["cpu_baseline"] = {"unavailable": str(e)}
    if rank == 0:
        print(json.dumps(out))
    if ws > 1:
        dist.destroy_process_group()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--rows", type=int, default=65536)
    p.add_argument("--cols", type=int, default=65536)
    p.add_argument("--e2e-iters", type=int, default=100)
    p.add_argument("--e2e-runs", type=int, default=2)
    p.add_argument("--e2e-pipeline", type=int, default=40, help="pipelined e2e steps (0: report the sequential e2e)")
    p.add_argument("--e2e-sets", type=int, default=3, help="array sets the pipelined e2e steps rotate over")
    p.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    p.add_argument("--cpu-rows", type=int, default=CPU_ROWS, help="rows of the heat CPU-baseline band (both arms)")
    p.add_argument("--cpu-iters", type=int, default=CPU_ITERS, help="timed launches of the main arm's heat CPU baseline")
    p.add_argument("--cpu-bounds-check", choices=["on", "off"], default="on",
                   help="--impl reference: the reference's array_view bounds checks (memory.hpp:54; default on, as shipped)")
    p.add_argument("--matmul-n", type=int, default=32768, help="C3 contraction size (0 to skip)")
    p.add_argument("--matmul-steps", type=int, default=5)
    p.add_argument("--tf32-steps", type=int, default=3, help="steps of the C3 fp32 (TF32) contraction leg (0 to skip)")
    p.add_argument("--no-c4", dest="c4", action="store_false", help="skip the histogram / k-means legs")
    p.add_argument("--hist-n", type=int, default=4_000_000_000)
    p.add_argument("--strip", type=int, default=128, help="N>1: rows of the halo-facing superblocks per GPU")
    p.add_argument("--km-n", type=int, default=1_000_000_000)
    p.add_argument("--no-c1", dest="c1", action="store_false", help="skip the BASELINE configs[0] leg (4096^2, 4 chunks)")
    p.add_argument("--nbody-n", type=int, default=65536, help="n-body leg (f64 all pairs, d=3); 0 to skip")
    p.add_argument("--c1-ref-iters", type=int, default=5)
    p.add_argument("--c1-strip", type=int, default=0, help="C1: rows of the halo-facing superblocks per chunk (0: one superblock per chunk)")
    p.add_argument("--ooc-gib", type=float, default=80.0, help="C5 out-of-core working set (2 arrays), 0 to skip")
    p.add_argument("--ooc-cap-gib", type=float, default=24.0, help="device capacity for the C5 leg (one array must not fit)")
    p.add_argument("--ooc-iters", type=int, default=12)
    args = p.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
