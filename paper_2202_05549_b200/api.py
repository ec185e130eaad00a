"""Host API mirroring the reference's driver / system_runtime / distribution interface.

Names and argument meaning follow proj/include/manta (planner.hpp:51-78 `driver`,
runtime.hpp:70-98 `system_runtime`, distribution.hpp:62-92 distributions); errors are the
reference's exception kinds (ParseError, ValidationError, PlanError, ExecutionError). All
work happens behind the C-ABI of include/manta_b200.h; this module only marshals.

`Context` combines the driver with its executor the way the reference's harnesses do
(test_runtime.cpp:12-43): `launch` plans, `flush` hands the new tasks to the executor
(take_pending + submit), `synchronize` waits.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from . import _capi as capi
from ._capi import (BF16, F32, F64, I32, I64, ExecutionError, MantaError, ParseError, PlanError,  # noqa: F401
                    ValidationError)

_NP_DTYPE = {I32: np.int32, I64: np.int64, F32: np.float32, F64: np.float64, BF16: np.uint16}


def dtype_code(t) -> int:
    if isinstance(t, str):
        return capi.DTYPE_NAMES[t]
    return int(t)


@dataclass(frozen=True)
class Chunk:
    id: int
    lo: tuple
    hi: tuple
    home: tuple  # (worker, device)


@dataclass(frozen=True)
class Superblock:
    lo: tuple
    hi: tuple
    device: tuple


@dataclass(frozen=True)
class Arr:
    """Launch argument naming a distributed array (launch_arg::array)."""
    id: int


def _devs(devices) -> tuple:
    arr = (capi.Device * max(1, len(devices)))()
    for i, (w, d) in enumerate(devices):
        arr[i].worker, arr[i].device = w, d
    return arr, len(devices)


def _chunks_out(lib, fn, *args) -> list[Chunk]:
    n = C.c_int64(0)
    lib.check(fn(*args, None, 0, C.byref(n)))
    buf = (capi.ChunkDesc * max(1, n.value))()
    lib.check(fn(*args, buf, n.value, C.byref(n)))
    return [Chunk(c.id, *c.region.box(), (c.home.worker, c.home.device)) for c in buf[: n.value]]


def _domain(domain) -> capi.Rect:
    if isinstance(domain, capi.Rect):
        return domain
    if len(domain) == 2 and isinstance(domain[0], (tuple, list)):
        return capi.Rect.make(domain[0], domain[1])
    return capi.Rect.make([0] * len(domain), domain)


class Distributions:
    """tile_data_dist / row_dist / col_dist / tile_dist / stencil_dist / replicated_dist /
    single_dist (distribution.cpp:136-195) and block_work_dist (:110-134)."""

    def __init__(self, lib: capi.Lib):
        self.lib = lib

    def tile_data(self, domain, extents, halo, devices, first_id=0) -> list[Chunk]:
        d = _domain(domain)
        ext = (C.c_int64 * 3)(*extents)
        hal = (C.c_int64 * 3)(*halo)
        devs, nd = _devs(devices)
        return _chunks_out(self.lib, self.lib.dist_tile, C.byref(d), ext, hal, devs, nd, first_id)

    def row(self, domain, rows, devices, first_id=0):
        d = _domain(domain)
        lo, hi = d.box()
        ext = [h - l for l, h in zip(lo, hi)]
        ext[0] = rows
        return self.tile_data(d, ext, [0] * d.rank, devices, first_id)

    def col(self, domain, cols, devices, first_id=0):
        d = _domain(domain)
        if d.rank < 2:
            raise ValidationError("column distribution requires rank >= 2")
        lo, hi = d.box()
        ext = [h - l for l, h in zip(lo, hi)]
        ext[1] = cols
        return self.tile_data(d, ext, [0] * d.rank, devices, first_id)

    def tile(self, domain, extents, devices, first_id=0):
        return self.tile_data(domain, extents, [0] * len(extents), devices, first_id)

    def stencil(self, domain, extents, halo, devices, first_id=0):
        return self.tile_data(domain, extents, halo, devices, first_id)

    def replicated(self, domain, devices, first_id=0):
        d = _domain(domain)
        devs, nd = _devs(devices)
        return _chunks_out(self.lib, self.lib.dist_replicated, C.byref(d), devs, nd, first_id)

    def single(self, domain, home, first_id=0):
        d = _domain(domain)
        dev = capi.Device(home[0], home[1])
        return _chunks_out(self.lib, self.lib.dist_single, C.byref(d), dev, first_id)

    def block_work(self, grid, block, threads_per_superblock, devices) -> list[Superblock]:
        g = _domain(grid)
        b = (C.c_int64 * 3)(*block)
        t = (C.c_int64 * 3)(*threads_per_superblock)
        devs, nd = _devs(devices)
        n = C.c_int64(0)
        self.lib.check(self.lib.work_block(C.byref(g), b, t, devs, nd, None, 0, C.byref(n)))
        out = (capi.Superblock * max(1, n.value))()
        self.lib.check(self.lib.work_block(C.byref(g), b, t, devs, nd, out, n.value, C.byref(n)))
        return [Superblock(*s.blocks.box(), (s.device.worker, s.device.device)) for s in out[: n.value]]


def _task_dict(t: capi.Task, pool, args) -> dict:
    d = {"id": t.id, "worker": t.worker, "kind": capi.TASK_KIND_NAMES[t.kind], "resource": (t.resource.worker, t.resource.device),
         "deps": [pool[t.deps_off + i] for i in range(t.ndeps)]}
    k = t.kind
    if k == capi.CREATE:
        d.update(chunk=t.chunk, region=t.region.box(), home=(t.home.worker, t.home.device), dtype=t.dtype, fill=t.fill,
                 fill_op=t.fill_op if t.fill == capi.FILL_IDENTITY else 0)
    elif k == capi.DELETE:
        d.update(chunk=t.chunk)
    elif k == capi.EXECUTE:
        d.update(kernel=t.kernel.decode(), device=(t.device.worker, t.device.device), sb_blocks=t.sb_blocks.box(),
                 sb_threads=t.sb_threads.box(), block_size=t.block_size.point(),
                 args=[(args[t.args_off + i].kind, args[t.args_off + i].i, args[t.args_off + i].f, args[t.args_off + i].chunk)
                       for i in range(t.nargs)])
    elif k == capi.COPY:
        d.update(src=t.src, dst=t.dst, src_region=t.src_region.box(), dst_region=t.dst_region.box())
    elif k in (capi.SEND, capi.RECV):
        d.update(chunk=t.chunk, region=t.region.box(), peer=t.peer, tag=t.tag)
    elif k == capi.REDUCE:
        d.update(op=t.op, inputs=[pool[t.inputs_off + i] for i in range(t.ninputs)], output=t.output)
    elif k in (capi.HOST_WRITE, capi.HOST_READ):
        d.update(chunk=t.chunk, region=t.region.box(), host_box=t.src_region.box(), host=t.tag, dtype=t.dtype)
    elif k == capi.ALLREDUCE:
        d.update(op=t.op, inputs=[pool[t.inputs_off + i] for i in range(t.ninputs)], output=t.output, tag=t.tag, region=t.region.box(),
                 dtype=t.dtype)
    return d


class PlanBuffer:
    """A flat task list + side pools, as exported by mt_plan_export / consumed by mt_exec_submit."""

    def __init__(self, tasks, pool, args):
        self.tasks, self.pool, self.args = tasks, pool, args

    def __len__(self):
        return len(self.tasks)

    def dicts(self) -> list[dict]:
        return [_task_dict(t, self.pool, self.args) for t in self.tasks]


def param_specs(params):
    """[(name, "scalar"|"array", dtype, rank, writable), ...] -> mt_param_spec array"""
    out = (capi.ParamSpec * max(1, len(params)))()
    for i, (name, kind, dt, rank, writable) in enumerate(params):
        out[i].name = name.encode()
        out[i].kind = capi.PARAM_ARRAY if kind == "array" else capi.PARAM_SCALAR
        out[i].dtype = capi.DTYPE_NAMES[dt]
        out[i].rank = int(rank)
        out[i].writable = int(bool(writable))
    return out


def wrapper_source(lib, kernel, params, block_offset, offsets, strides) -> str:
    """The wrapper text one superblock instance compiles to (reference generate_wrapper_source,
    kernels.cpp:540-596); offsets/strides: one list per array parameter."""
    spec = param_specs(params)
    bo = (C.c_int64 * max(1, len(block_offset)))(*block_offset)
    flat_o = [v for o in offsets for v in o]
    flat_s = [v for s_ in strides for v in s_]
    o = (C.c_int64 * max(1, len(flat_o)))(*flat_o)
    st = (C.c_int64 * max(1, len(flat_s)))(*flat_s)
    n = C.c_int64(0)
    lib.check(lib.wrapper_source(kernel.encode(), spec, len(params), bo, len(block_offset), o, st, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    lib.check(lib.wrapper_source(kernel.encode(), spec, len(params), bo, len(block_offset), o, st, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def _nccl_library():
    """torch's bundled libnccl.so.2 (the one torch.distributed uses), else None (default search)"""
    try:
        import nvidia.nccl
        path = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
        return path.encode() if os.path.exists(path) else None
    except ImportError:
        return None


class Context:
    """driver + executor over one library (product `mt_` or oracle shim `mr_`)."""

    def __init__(self, lib: capi.Lib, workers=1, devices=1, execute=True, compat_deps=False, suppress_conflict_deps=False,
                 num_gpus=0, streams_per_device=0, device_capacity=0, host_capacity=0, staging_threshold=0, record_accesses=False,
                 lookahead_tasks=0, worker_rank=None, gpu_base=0, collective_reduce=False, retain_plan=True, disk_capacity=0,
                 spill_dir=None, schedule_seed=0, plan_cache=True):
        self.lib = lib
        self.dist = Distributions(lib)
        cfg = capi.Config()
        cfg.workers, cfg.devices_per_worker = workers, devices
        cfg.suppress_conflict_deps = int(suppress_conflict_deps)
        cfg.compat_deps = int(compat_deps)
        cfg.execute = int(execute)
        cfg.num_gpus = num_gpus
        cfg.streams_per_device = streams_per_device
        cfg.device_capacity = device_capacity
        cfg.host_capacity = host_capacity
        cfg.staging_threshold = staging_threshold
        cfg.record_accesses = int(record_accesses)
        cfg.lookahead_tasks = int(lookahead_tasks)
        cfg.collective_reduce = int(collective_reduce)
        cfg.drop_executed_tasks = int(not retain_plan)  # long runs: forget tasks once queued
        cfg.disk_capacity = int(disk_capacity)
        self._spill_dir = spill_dir.encode() if spill_dir else None
        cfg.spill_dir = self._spill_dir
        cfg.schedule_seed = int(schedule_seed)
        cfg.plan_cache_off = int(not plan_cache)
        if worker_rank is not None:  # one process per worker
            cfg.single_worker, cfg.worker_rank, cfg.gpu_base = 1, int(worker_rank), int(gpu_base)
        self.single_worker = worker_rank is not None
        self.collective_reduce = bool(collective_reduce)
        h = C.c_void_p()
        lib.check(lib.ctx_create(C.byref(cfg), C.byref(h)))
        self.h = h
        self.executes = bool(execute)
        self._arrays: dict[int, tuple] = {}
        self._inflight: list = []  # host buffers of queued async transfers
        self._work_cache: dict = {}
        self._call_cache: dict = {}

    def close(self):
        if self.h:
            self.lib.check(self.lib.ctx_destroy(self.h))
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- driver ------------------------------------------------------------------------
    @property
    def devices(self) -> list[tuple]:
        out = (capi.Device * 4096)()
        n = C.c_int32(0)
        self.lib.check(self.lib.ctx_devices(self.h, out, 4096, C.byref(n)))
        return [(d.worker, d.device) for d in out[: n.value]]

    def create_array(self, domain, dtype, distribution: Sequence[Chunk], fill=None) -> int:
        d = _domain(domain)
        chunks = (capi.ChunkDesc * len(distribution))()
        for i, c in enumerate(distribution):
            chunks[i].id = c.id
            chunks[i].region = capi.Rect.make(c.lo, c.hi)
            chunks[i].home = capi.Device(*c.home)
        fill_code = {None: capi.FILL_NONE, 0: capi.FILL_ZERO, 0.0: capi.FILL_ZERO, 1: capi.FILL_ONE, 1.0: capi.FILL_ONE}[fill]
        out = C.c_int64(-1)
        self.lib.check(self.lib.array_create(self.h, C.byref(d), dtype_code(dtype), chunks, len(distribution), fill_code, C.byref(out)))
        self._arrays[out.value] = (d.box(), dtype_code(dtype))
        return out.value

    def delete_array(self, array_id: int):
        self.lib.check(self.lib.array_delete(self.h, array_id))

    def chunks(self, array_id: int) -> list[Chunk]:
        return _chunks_out(self.lib, self.lib.array_chunks, self.h, array_id)

    def launch(self, kernel: str, grid, block, work: Sequence[Superblock], args: Iterable, annotation: str):
        args = list(args)
        # iterative launches repeat one call: its ctypes structures are converted once (the type
        # is part of the key so that 1, 1.0 and True stay distinct arguments)
        try:
            ckey = (kernel, tuple(grid) if not isinstance(grid, capi.Rect) else None, tuple(block), tuple(work),
                    tuple((type(a), a) for a in args), annotation)
            hit = self._call_cache.get(ckey) if ckey[1] is not None else None
        except TypeError:  # unhashable argument: convert without caching
            ckey, hit = None, None
        if hit is None:
            hit = self._convert_launch(kernel, grid, block, work, args, annotation)
            if ckey is not None and ckey[1] is not None:
                if len(self._call_cache) > 64:
                    self._call_cache.clear()
                self._call_cache[ckey] = hit
        kb, g, b, w, nw, la, na, ab = hit
        first, last = C.c_int64(0), C.c_int64(0)
        self.lib.check(self.lib.launch(self.h, kb, C.byref(g), b, w, nw, la, na, ab, C.byref(first), C.byref(last)))
        return first.value, last.value

    def launch_repeat(self, kernel: str, grid, block, work: Sequence[Superblock], args: Iterable, annotation: str, repeat: int,
                      swap=None, flush_every=0):
        """`repeat` launches of one request in a single call (the repeat loop of apply_scenario,
        scenario.cpp:407-441): after each launch the array arguments `swap` = (a, b) exchange
        roles (the scenario's name swap); tasks go to the executor every `flush_every` launches
        (0: at the end). Returns the task id range of all launches."""
        kb, g, b, w, nw, la, na, ab = self._convert_launch(kernel, grid, block, work, list(args), annotation)
        sa, sb = (-1, -1) if swap is None else (int(getattr(swap[0], "id", swap[0])), int(getattr(swap[1], "id", swap[1])))
        first, last = C.c_int64(0), C.c_int64(0)
        self.lib.check(self.lib.launch_repeat(self.h, kb, C.byref(g), b, w, nw, la, na, ab, int(repeat), sa, sb, int(flush_every), C.byref(first),
                                              C.byref(last)))
        return first.value, last.value

    def _convert_launch(self, kernel, grid, block, work, args, annotation):
        g = _domain(grid)
        b = (C.c_int64 * 3)(*block)
        key = tuple(work)  # iterative launches reuse one decomposition: convert it once
        w = self._work_cache.get(key)
        if w is None:
            w = (capi.Superblock * max(1, len(work)))()
            for i, s in enumerate(work):
                w[i].blocks = capi.Rect.make(s.lo, s.hi)
                w[i].device = capi.Device(*s.device)
            if len(self._work_cache) > 64:
                self._work_cache.clear()
            self._work_cache[key] = w
        la = (capi.LaunchArg * max(1, len(args)))()
        for i, a in enumerate(args):
            if isinstance(a, Arr):
                la[i].kind, la[i].array = capi.LARG_ARRAY, a.id
            elif isinstance(a, (bool, int, np.integer)):
                la[i].kind, la[i].i = capi.LARG_INT, int(a)
            elif isinstance(a, (float, np.floating)):
                la[i].kind, la[i].f = capi.LARG_FLOAT, float(a)
            else:
                raise ValidationError(f"unsupported launch argument {a!r}")
        return kernel.encode(), g, b, w, len(work), la, len(args), annotation.encode()

    def flush(self):
        self.lib.check(self.lib.flush(self.h))

    def synchronize(self):
        self.lib.check(self.lib.sync(self.h))
        self._inflight.clear()

    # -- data ------------------------------------------------------------------------
    def shape_of(self, array_id: int):
        (lo, hi), t = self._arrays[array_id]
        return tuple(h - l for l, h in zip(lo, hi)), t

    def read(self, array_id: int) -> np.ndarray:
        shape, t = self.shape_of(array_id)
        out = np.empty(shape, dtype=_NP_DTYPE[t])
        self.lib.check(self.lib.array_read(self.h, array_id, out.ctypes.data, out.nbytes))
        return out

    def write(self, array_id: int, data: np.ndarray):
        shape, t = self.shape_of(array_id)
        data = np.ascontiguousarray(data, dtype=_NP_DTYPE[t]).reshape(shape)
        self.lib.check(self.lib.array_write(self.h, array_id, data.ctypes.data, data.nbytes))

    # -- runtime-compiled kernels -----------------------------------
    def compile_kernel(self, kernel: str, params, source: str) -> None:
        """Register `source` (a __device__ function named `kernel` taking the virtual block
        index first, then `params` in order) for this context; compiled with NVRTC for
        sm_100a now (errors raise ValidationError with the compiler log) and per superblock
        instance on first launch."""
        self.lib.check(self.lib.ctx_kernel_compile(self.h, kernel.encode(), param_specs(params), len(params), source.encode()))

    # -- asynchronous host transfers (planned as tasks; see mt_array_write_async) ---------
    def write_async(self, array_id: int, data, box=None) -> None:
        """Queue an upload of `data` (C-contiguous, the array's shape and dtype; numpy or a
        pinned torch tensor) into every chunk. The buffer must stay untouched until
        synchronize(); the context keeps a reference until then. With `box` = (lo, hi) the
        buffer holds only that box of the array (one process per GPU: each rank passes its
        own chunks' box; mt_array_write_box_async)."""
        ptr, nbytes = self._host_buffer(array_id, data, box)
        if box is None:
            self.lib.check(self.lib.array_write_async(self.h, array_id, ptr, nbytes))
        else:
            r = capi.Rect.make(*box)
            self.lib.check(self.lib.array_write_box_async(self.h, array_id, C.byref(r), ptr, nbytes))
        self._inflight.append(data)

    def read_async(self, array_id: int, out, box=None) -> None:
        """Queue a download of the array into `out` (C-contiguous, the array's shape and dtype,
        or the shape of `box`); valid after synchronize()."""
        ptr, nbytes = self._host_buffer(array_id, out, box)
        if box is None:
            self.lib.check(self.lib.array_read_async(self.h, array_id, ptr, nbytes))
        else:
            r = capi.Rect.make(*box)
            self.lib.check(self.lib.array_read_box_async(self.h, array_id, C.byref(r), ptr, nbytes))
        self._inflight.append(out)

    def _host_buffer(self, array_id, buf, box=None):
        shape, t = self.shape_of(array_id)
        if box is not None:
            shape = [h - l for l, h in zip(*box)]
        if isinstance(buf, np.ndarray):
            if not buf.flags["C_CONTIGUOUS"] or buf.dtype != np.dtype(_NP_DTYPE[t]) or list(buf.shape) != list(shape):
                raise ValidationError("host buffer must be C-contiguous with the array's (or the box's) shape and dtype")
            return buf.ctypes.data, buf.nbytes
        # torch tensor (e.g. pinned host memory)
        if buf.is_cuda or not buf.is_contiguous() or list(buf.shape) != list(shape):
            raise ValidationError("host buffer must be a contiguous host tensor with the array's (or the box's) shape")
        import torch
        want = {I32: (torch.int32,), I64: (torch.int64,), F32: (torch.float32,), F64: (torch.float64,),
                BF16: (torch.bfloat16, torch.uint16, torch.int16)}[t]
        if buf.dtype not in want:
            raise ValidationError(f"host tensor dtype {buf.dtype} does not match the array's element type { {v: k for k, v in capi.DTYPE_NAMES.items()}.get(t, t)}")
        return buf.data_ptr(), buf.numel() * buf.element_size()

    def replicas_coherent(self, array_id: int) -> bool:
        ok = C.c_int32(0)
        self.lib.check(self.lib.array_check_replicas(self.h, array_id, C.byref(ok)))
        return bool(ok.value)

    # -- plan --------------------------------------------------------------------------
    def plan_size(self) -> int:
        return int(self.lib.plan_size(self.h))

    def plan_cache_hits(self) -> int:
        return int(self.lib.plan_cache_hits(self.h)) if self.lib.has("plan_cache_hits") else 0

    def export_plan(self, first=0, last=None) -> PlanBuffer:
        if last is None:
            last = 1 << 62
        nt, npool, na = C.c_int64(0), C.c_int64(0), C.c_int64(0)
        self.lib.check(self.lib.plan_export(self.h, first, last, None, 0, C.byref(nt), None, 0, C.byref(npool), None, 0, C.byref(na)))
        tasks = (capi.Task * max(1, nt.value))()
        pool = (C.c_int64 * max(1, npool.value))()
        args = (capi.ArgBinding * max(1, na.value))()
        self.lib.check(self.lib.plan_export(self.h, first, last, tasks, nt.value, C.byref(nt), pool, npool.value, C.byref(npool), args, na.value,
                                            C.byref(na)))
        return PlanBuffer(tasks[: nt.value], pool, args)

    def plan(self, first=0, last=None) -> list[dict]:
        return self.export_plan(first, last).dicts()

    def accesses(self) -> list[tuple]:
        """(task, chunk, (lo, hi), write) for every planned access of a non-temporary chunk."""
        n = C.c_int64(0)
        self.lib.check(self.lib.plan_accesses(self.h, None, 0, C.byref(n)))
        buf = (capi.Access * max(1, n.value))()
        self.lib.check(self.lib.plan_accesses(self.h, buf, n.value, C.byref(n)))
        return [(a.task, a.chunk, a.region.box(), bool(a.write)) for a in buf[: n.value]]

    def chunk_meta(self, chunk: int):
        desc = capi.ChunkDesc()
        dt, tmp = C.c_int32(0), C.c_int32(0)
        self.lib.check(self.lib.chunk_meta(self.h, chunk, C.byref(desc), C.byref(dt), C.byref(tmp)))
        return Chunk(desc.id, *desc.region.box(), (desc.home.worker, desc.home.device)), dt.value, bool(tmp.value)

    def exec_stats(self) -> dict:
        ex = self.lib.ctx_exec(self.h)
        if not ex or not self.lib.has("exec_stats"):
            return {}
        keys = ["tasks", "kernels", "copies", "bytes_copied", "bytes_sent", "bytes_received", "peak_device_bytes", "evictions",
                "spill_bytes_d2h", "spill_bytes_h2d", "dead_drops", "dead_skips", "host_reclaims",
                "host_write_bytes", "host_read_bytes", "graph_captures", "graph_replays", "bytes_host_to_disk", "bytes_disk_to_host", "messages", "message_ops",
                "fused_copies", "bytes_fused"]
        out = (C.c_uint64 * len(keys))()
        self.lib.check(self.lib.exec_stats(ex, out, len(keys)))
        return dict(zip(keys, [int(v) for v in out]))

    def report_json(self) -> str:
        """run_report::to_json of the attached executor (runtime.cpp:613-636)"""
        ex = self._ex()
        n = C.c_int64(0)
        self.lib.check(self.lib.exec_report_json(ex, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self.lib.check(self.lib.exec_report_json(ex, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    # -- one process per worker ------------------------------------------------------
    def peer_export(self) -> bytes:
        n = C.c_int64(0)
        self.lib.check(self.lib.ctx_peer_export(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        self.lib.check(self.lib.ctx_peer_export(self.h, buf, n.value, C.byref(n)))
        return buf.raw[: n.value]

    def peer_import(self, blobs: Sequence[bytes]):
        size = len(blobs[0])
        if any(len(b) != size for b in blobs):
            raise ValidationError("mailbox blobs differ in size")
        data = b"".join(blobs)
        self.lib.check(self.lib.ctx_peer_import(self.h, data, size, len(blobs)))

    def connect_peers(self, group=None):
        """Exchange mailboxes with every rank of the torch.distributed group and map them; with
        collective_reduce also create the NCCL communicator the allreduce tasks run on."""
        import torch.distributed as dist
        mine = self.peer_export()
        blobs = [None] * dist.get_world_size(group)
        dist.all_gather_object(blobs, mine, group=group)
        self.peer_import(blobs)
        if self.collective_reduce and self.single_worker:
            lib = _nccl_library()
            ident = [None]
            if dist.get_rank(group) == 0:
                buf = C.create_string_buffer(128)
                self.lib.check(self.lib.ctx_nccl_unique_id(self.h, lib, buf))
                ident[0] = buf.raw
            dist.broadcast_object_list(ident, src=0, group=group)
            self.lib.check(self.lib.ctx_nccl_init(self.h, lib, ident[0]))

    # -- device timing (bench) ------------------------------------------------------
    def _ex(self):
        ex = self.lib.ctx_exec(self.h)
        if not ex:
            raise ValidationError("context does not execute")
        return ex

    def mark(self, slot: int):
        """Device event completing when all work enqueued so far has completed (0=start, 1=stop)."""
        self.flush()
        self.lib.check(self.lib.exec_mark(self._ex(), slot))

    def elapsed_ms(self) -> float:
        v = C.c_double(0)
        self.lib.check(self.lib.exec_elapsed_ms(self._ex(), C.byref(v)))
        return v.value

    def profile_kernels(self, on=True):
        self.lib.check(self.lib.exec_profile(self._ex(), int(on)))

    def trace(self, on=True):
        """per-task device timestamps in report_json() (mt_exec_trace)"""
        self.lib.check(self.lib.exec_trace(self._ex(), int(on)))

    def kernel_time(self, kernel: str) -> tuple[int, float]:
        n, ms = C.c_int64(0), C.c_double(0)
        self.lib.check(self.lib.exec_kernel_time(self._ex(), kernel.encode(), C.byref(n), C.byref(ms)))
        return n.value, ms.value

    def last_stream(self) -> int:
        ex = self.lib.ctx_exec(self.h)
        return int(self.lib.exec_last_stream(ex) or 0) if ex and self.lib.has("exec_last_stream") else 0


class Executor:
    """system_runtime alone: consumes flat plans (e.g. the reference driver's) — the drop-in
    path for the reference's CPU executor (runtime.hpp:70-98)."""

    def __init__(self, lib: capi.Lib, workers=1, devices=1, num_gpus=0, device_capacity=0):
        self.lib = lib
        cfg = capi.Config()
        cfg.workers, cfg.devices_per_worker, cfg.execute, cfg.num_gpus = workers, devices, 1, num_gpus
        cfg.device_capacity = device_capacity
        h = C.c_void_p()
        lib.check(lib.exec_create(C.byref(cfg), C.byref(h)))
        self.h = h

    def submit(self, plan: PlanBuffer):
        if len(plan) == 0:
            return
        arr = (capi.Task * len(plan.tasks))(*plan.tasks)
        self.lib.check(self.lib.exec_submit(self.h, arr, len(plan.tasks), plan.pool, plan.args))

    def synchronize(self):
        self.lib.check(self.lib.exec_sync(self.h))

    def read_chunk(self, chunk: int, nbytes: int) -> bytes:
        buf = (C.c_char * nbytes)()
        self.lib.check(self.lib.exec_read_chunk(self.h, chunk, buf, nbytes))
        return bytes(buf)

    def report_json(self) -> str:
        n = C.c_int64(0)
        self.lib.check(self.lib.exec_report_json(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self.lib.check(self.lib.exec_report_json(self.h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def close(self):
        if self.h:
            self.lib.check(self.lib.exec_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
