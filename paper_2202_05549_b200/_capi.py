"""ctypes mirror of include/manta_b200.h.

`Lib(path, prefix)` binds every entry point of the C-ABI. The product library
(libmanta_b200.so, prefix ``mt_``) and the oracle shim over the unmodified reference
(oracle/_ref/libmanta_ref.so, prefix ``mr_``; test infrastructure only) export the same
functions, so one binding drives both.
"""
from __future__ import annotations

import ctypes as C

MAX_RANK = 3
KERNEL_NAME_MAX = 64

# status codes (errors.hpp:9-35)
MT_OK, MT_EPARSE, MT_EVALIDATION, MT_EPLAN, MT_EEXEC, MT_EINTERNAL = range(6)
# dtypes (dtype.hpp:13 + bf16)
I32, I64, F32, F64, BF16 = range(5)
DTYPE_NAMES = {"i32": I32, "i64": I64, "f32": F32, "f64": F64, "bf16": BF16}
DTYPE_SIZE = {I32: 4, I64: 8, F32: 4, F64: 8, BF16: 2}
# task kinds (task.hpp:32-95)
CREATE, DELETE, EXECUTE, COPY, SEND, RECV, REDUCE, ALLREDUCE, HOST_WRITE, HOST_READ = range(10)
TASK_KIND_NAMES = ["create", "delete", "execute", "copy", "send", "recv", "reduce", "allreduce", "host_write", "host_read"]
FILL_NONE, FILL_ZERO, FILL_ONE, FILL_IDENTITY = range(4)
RED_PLUS, RED_TIMES, RED_MIN, RED_MAX = range(4)
ARG_INT, ARG_FLOAT, ARG_CHUNK, ARG_NONE = range(4)
LARG_INT, LARG_FLOAT, LARG_ARRAY = range(3)
PARAM_SCALAR, PARAM_ARRAY = range(2)


class Rect(C.Structure):
    _fields_ = [("rank", C.c_int32), ("pad_", C.c_int32), ("lo", C.c_int64 * MAX_RANK), ("hi", C.c_int64 * MAX_RANK)]

    @classmethod
    def make(cls, lo, hi=None):
        r = cls()
        r.rank = len(lo)
        for k, v in enumerate(lo):
            r.lo[k] = int(v)
        if hi is not None:
            for k, v in enumerate(hi):
                r.hi[k] = int(v)
        return r

    def box(self):
        return (tuple(self.lo[: self.rank]), tuple(self.hi[: self.rank]))

    def point(self):
        return tuple(self.lo[: self.rank])


class Device(C.Structure):
    _fields_ = [("worker", C.c_int32), ("device", C.c_int32)]


class ChunkDesc(C.Structure):
    _fields_ = [("id", C.c_int64), ("region", Rect), ("home", Device)]


class Superblock(C.Structure):
    _fields_ = [("blocks", Rect), ("device", Device)]


class ArgBinding(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("i", C.c_int64), ("f", C.c_double), ("chunk", C.c_int64)]


class Task(C.Structure):
    _fields_ = [
        ("id", C.c_int64), ("worker", C.c_int32), ("kind", C.c_int32), ("resource", Device),
        ("deps_off", C.c_int64), ("ndeps", C.c_int64),
        ("chunk", C.c_int64), ("region", Rect), ("home", Device),
        ("dtype", C.c_int32), ("fill", C.c_int32), ("fill_op", C.c_int32), ("op", C.c_int32),
        ("kernel", C.c_char * KERNEL_NAME_MAX), ("device", Device),
        ("sb_blocks", Rect), ("sb_threads", Rect), ("block_size", Rect),
        ("args_off", C.c_int64), ("nargs", C.c_int64),
        ("src", C.c_int64), ("dst", C.c_int64), ("src_region", Rect), ("dst_region", Rect),
        ("peer", C.c_int32), ("pad_", C.c_int32), ("tag", C.c_uint64),
        ("inputs_off", C.c_int64), ("ninputs", C.c_int64), ("output", C.c_int64),
    ]


class LaunchArg(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("i", C.c_int64), ("f", C.c_double), ("array", C.c_int64)]


class Config(C.Structure):
    _fields_ = [
        ("workers", C.c_int32), ("devices_per_worker", C.c_int32), ("suppress_conflict_deps", C.c_int32),
        ("compat_deps", C.c_int32), ("execute", C.c_int32), ("num_gpus", C.c_int32),
        ("streams_per_device", C.c_int32), ("single_worker", C.c_int32),
        ("device_capacity", C.c_uint64), ("host_capacity", C.c_uint64), ("staging_threshold", C.c_uint64),
        ("record_accesses", C.c_int32), ("lookahead_tasks", C.c_int32),
        ("worker_rank", C.c_int32), ("gpu_base", C.c_int32), ("collective_reduce", C.c_int32), ("drop_executed_tasks", C.c_int32), ("disk_capacity", C.c_uint64), ("spill_dir", C.c_char_p),
        ("schedule_seed", C.c_uint64), ("plan_cache_off", C.c_int32), ("pad_", C.c_int32),
    ]


class Access(C.Structure):
    _fields_ = [("task", C.c_int64), ("chunk", C.c_int64), ("region", Rect), ("write", C.c_int32), ("pad_", C.c_int32)]


class View(C.Structure):
    _fields_ = [("base", C.c_void_p), ("dtype", C.c_int32), ("rank", C.c_int32), ("offset", C.c_int64 * MAX_RANK),
                ("stride", C.c_int64 * MAX_RANK), ("extent", C.c_int64 * MAX_RANK)]


class LaunchCtx(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nparams", C.c_int32), ("block_offset", C.c_int64 * MAX_RANK),
                ("block_count", C.c_int64 * MAX_RANK), ("block_size", C.c_int64 * MAX_RANK),
                ("threads_lo", C.c_int64 * MAX_RANK), ("threads_hi", C.c_int64 * MAX_RANK),
                ("scalars_int", C.POINTER(C.c_int64)), ("scalars_float", C.POINTER(C.c_double)),
                ("views", C.POINTER(View)), ("user", C.c_void_p), ("nmirrors", C.c_int32),
                ("mirrors", C.c_void_p), ("mirror_applied", C.POINTER(C.c_int32))]


class Mirror(C.Structure):
    _fields_ = [("param", C.c_int32), ("pad_", C.c_int32), ("lo", C.c_int64 * MAX_RANK), ("hi", C.c_int64 * MAX_RANK), ("dst", View)]


class ParamSpec(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("kind", C.c_int32), ("dtype", C.c_int32), ("rank", C.c_int32), ("writable", C.c_int32)]


LAUNCHER = C.CFUNCTYPE(C.c_int, C.POINTER(LaunchCtx), C.c_void_p)

P = C.POINTER
_SIGS = {
    "last_error": (C.c_char_p, []),
    "version": (C.c_char_p, []),
    "dist_tile": (C.c_int, [P(Rect), P(C.c_int64), P(C.c_int64), P(Device), C.c_int32, C.c_int64, P(ChunkDesc), C.c_int64, P(C.c_int64)]),
    "dist_replicated": (C.c_int, [P(Rect), P(Device), C.c_int32, C.c_int64, P(ChunkDesc), C.c_int64, P(C.c_int64)]),
    "dist_single": (C.c_int, [P(Rect), Device, C.c_int64, P(ChunkDesc), C.c_int64, P(C.c_int64)]),
    "work_block": (C.c_int, [P(Rect), P(C.c_int64), P(C.c_int64), P(Device), C.c_int32, P(Superblock), C.c_int64, P(C.c_int64)]),
    "ctx_create": (C.c_int, [P(Config), P(C.c_void_p)]),
    "ctx_destroy": (C.c_int, [C.c_void_p]),
    "ctx_devices": (C.c_int, [C.c_void_p, P(Device), C.c_int32, P(C.c_int32)]),
    "array_create": (C.c_int, [C.c_void_p, P(Rect), C.c_int32, P(ChunkDesc), C.c_int64, C.c_int32, P(C.c_int64)]),
    "array_delete": (C.c_int, [C.c_void_p, C.c_int64]),
    "array_chunks": (C.c_int, [C.c_void_p, C.c_int64, P(ChunkDesc), C.c_int64, P(C.c_int64)]),
    "launch": (C.c_int, [C.c_void_p, C.c_char_p, P(Rect), P(C.c_int64), P(Superblock), C.c_int64, P(LaunchArg), C.c_int32, C.c_char_p,
                         P(C.c_int64), P(C.c_int64)]),
    "launch_repeat": (C.c_int, [C.c_void_p, C.c_char_p, P(Rect), P(C.c_int64), P(Superblock), C.c_int64, P(LaunchArg), C.c_int32, C.c_char_p,
                                C.c_int32, C.c_int64, C.c_int64, C.c_int32, P(C.c_int64), P(C.c_int64)]),
    "flush": (C.c_int, [C.c_void_p]),
    "sync": (C.c_int, [C.c_void_p]),
    "array_read": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_uint64]),
    "array_write": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_uint64]),
    "array_check_replicas": (C.c_int, [C.c_void_p, C.c_int64, P(C.c_int32)]),
    "plan_export": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, P(Task), C.c_int64, P(C.c_int64), P(C.c_int64), C.c_int64, P(C.c_int64),
                              P(ArgBinding), C.c_int64, P(C.c_int64)]),
    "plan_size": (C.c_int64, [C.c_void_p]),
    "plan_cache_hits": (C.c_uint64, [C.c_void_p]),
    "plan_accesses": (C.c_int, [C.c_void_p, P(Access), C.c_int64, P(C.c_int64)]),
    "chunk_meta": (C.c_int, [C.c_void_p, C.c_int64, P(ChunkDesc), P(C.c_int32), P(C.c_int32)]),
    "ctx_exec": (C.c_void_p, [C.c_void_p]),
    "exec_create": (C.c_int, [P(Config), P(C.c_void_p)]),
    "exec_destroy": (C.c_int, [C.c_void_p]),
    "exec_submit": (C.c_int, [C.c_void_p, P(Task), C.c_int64, P(C.c_int64), P(ArgBinding)]),
    "exec_sync": (C.c_int, [C.c_void_p]),
    "exec_read_chunk": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_uint64]),
    "exec_write_chunk": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_uint64]),
    "exec_report_json": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64, P(C.c_int64)]),
    "exec_stats": (C.c_int, [C.c_void_p, P(C.c_uint64), C.c_int32]),
    "exec_last_stream": (C.c_void_p, [C.c_void_p]),
    "exec_mark": (C.c_int, [C.c_void_p, C.c_int32]),
    "exec_elapsed_ms": (C.c_int, [C.c_void_p, P(C.c_double)]),
    "exec_profile": (C.c_int, [C.c_void_p, C.c_int32]),
    "exec_trace": (C.c_int, [C.c_void_p, C.c_int32]),
    "exec_kernel_time": (C.c_int, [C.c_void_p, C.c_char_p, P(C.c_int64), P(C.c_double)]),
    "kernel_register": (C.c_int, [C.c_char_p, P(ParamSpec), C.c_int32, LAUNCHER]),
    "kernel_count": (C.c_int, []),
    "ctx_kernel_register": (C.c_int, [C.c_void_p, C.c_char_p, P(ParamSpec), C.c_int32, C.c_void_p, C.c_void_p]),
    "ctx_gather_register": (C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int32, P(C.c_int32), P(Rect)]),
    "ctx_peer_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, P(C.c_int64)]),
    "ctx_peer_import": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32]),
    "ctx_nccl_unique_id": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p]),
    "array_write_async": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_uint64]),
    "ctx_kernel_compile": (C.c_int, [C.c_void_p, C.c_char_p, P(ParamSpec), C.c_int32, C.c_char_p]),
    "wrapper_source": (C.c_int, [C.c_char_p, P(ParamSpec), C.c_int32, P(C.c_int64), C.c_int32, P(C.c_int64), P(C.c_int64), C.c_char_p, C.c_int64,
                                 P(C.c_int64)]),
    "array_write_box_async": (C.c_int, [C.c_void_p, C.c_int64, P(Rect), C.c_void_p, C.c_uint64]),
    "array_read_box_async": (C.c_int, [C.c_void_p, C.c_int64, P(Rect), C.c_void_p, C.c_uint64]),
    "array_read_async": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_uint64]),
    "ctx_nccl_init": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p]),
    "fuzz_scenario_json": (C.c_int, [C.c_uint64, C.c_char_p, C.c_int64, P(C.c_int64)]),
    "scenario_plan": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P(Task), C.c_int64, P(C.c_int64), P(C.c_int64),
                                C.c_int64, P(C.c_int64), P(ArgBinding), C.c_int64, P(C.c_int64)]),
    "scenario_dot": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.c_char_p, C.c_int64, P(C.c_int64)]),
    "scenario_run": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_void_p, C.c_int64, P(C.c_int64),
                               P(C.c_int32)]),
    "kernel_info": (C.c_int, [C.c_int32, C.c_char_p, C.c_int32, P(ParamSpec), C.c_int32, P(C.c_int32)]),
    "annotation_describe": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int64, P(C.c_int64)]),
}
# entry points the oracle shim may lack
_OPTIONAL = {"exec_stats", "exec_last_stream", "kernel_info", "host_threads", "ctx_kernel_register", "fuzz_scenario_json", "scenario_plan", "scenario_dot",
             "scenario_run", "plan_accesses", "ctx_gather_register", "ctx_peer_export", "ctx_peer_import", "ctx_nccl_unique_id", "ctx_nccl_init", "array_write_async", "array_read_async", "array_write_box_async", "array_read_box_async", "ctx_kernel_compile", "wrapper_source", "exec_mark", "exec_elapsed_ms", "exec_profile", "exec_kernel_time", "exec_trace",
             "plan_cache_hits"}


class MantaError(RuntimeError):
    """Base of the reference's exception hierarchy (errors.hpp:9-35)."""


class ParseError(MantaError):
    pass


class ValidationError(MantaError):
    pass


class PlanError(MantaError):
    pass


class ExecutionError(MantaError):
    pass


_ERRORS = {MT_EPARSE: ParseError, MT_EVALIDATION: ValidationError, MT_EPLAN: PlanError, MT_EEXEC: ExecutionError}


class Lib:
    """Bound C-ABI of one library (product or oracle shim)."""

    def __init__(self, path: str, prefix: str):
        self.path = path
        self.prefix = prefix
        self.dll = C.CDLL(path)  # RTLD_LOCAL: product and oracle shim must never interpose
        for name, (res, args) in _SIGS.items():
            sym = prefix + name
            if not hasattr(self.dll, sym):
                if name in _OPTIONAL:
                    continue
                raise ImportError(f"{path} does not export {sym}")
            fn = getattr(self.dll, sym)
            fn.restype = res
            fn.argtypes = args
            setattr(self, name, fn)

    def check(self, rc: int):
        if rc == MT_OK:
            return
        msg = self.last_error().decode(errors="replace")
        raise _ERRORS.get(rc, MantaError)(msg)

    def has(self, name: str) -> bool:
        return hasattr(self, name)
