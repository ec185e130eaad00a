"""B200-native distributed kernel launches over annotated, chunked arrays.

A from-scratch implementation of the data-parallel hot path of Lightning
(arXiv 2202.05549; reference: /root/reference/proj, "manta"): the annotation-driven planner,
the HBM chunk store, the stream/event GPU executor, NVLink data movement and the sm_100a
benchmark kernels, all native (C++ / CUDA) behind the C-ABI in include/manta_b200.h.

There is no CPU fallback: the product library must be built (``__graft_entry__.build()``)
and executing contexts need a CUDA device; both fail loudly otherwise.
"""
from __future__ import annotations

import os

from . import _capi
from .api import Arr, Chunk, Context, Distributions, Executor, Superblock  # noqa: F401
from ._capi import ExecutionError, MantaError, ParseError, PlanError, ValidationError  # noqa: F401

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmanta_b200.so")

_lib = None


def lib() -> _capi.Lib:
    """The product C-ABI (libmanta_b200.so, prefix mt_)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        _lib = _capi.Lib(LIB_PATH, "mt_")
    return _lib


def context(**kw) -> Context:
    return Context(lib(), **kw)
