"""ORACLE / TEST INFRASTRUCTURE: the reference's own run_scenario and plan through the oracle
shim (oracle/_ref, prefix mr_), returning the same structures as the product's
paper_2202_05549_b200.scenario helpers. Used by tests/ and oracle/make_golden.py only."""
from __future__ import annotations

import json

import numpy as np

from paper_2202_05549_b200 import _capi as capi
from paper_2202_05549_b200.api import _NP_DTYPE


def run(ref_lib: capi.Lib, sc: dict, workers=0, devices=0, oracle_mode=True, ready_seed=None) -> tuple[dict, bool]:
    """The reference's own run_scenario (through the oracle shim)."""
    import ctypes as C
    text = json.dumps(sc).encode()
    n, coh = C.c_int64(0), C.c_int32(0)
    seed = 0 if ready_seed is None else ready_seed
    ref_lib.check(ref_lib.scenario_run(text, workers, devices, int(oracle_mode), seed, int(ready_seed is not None), None, 0, C.byref(n), C.byref(coh)))
    buf = np.empty(n.value, dtype=np.uint8)
    ref_lib.check(ref_lib.scenario_run(text, workers, devices, int(oracle_mode), seed, int(ready_seed is not None), buf.ctypes.data, n.value,
                                       C.byref(n), C.byref(coh)))
    out, off = {}, 0
    for a in sc.get("arrays", []):
        t = capi.DTYPE_NAMES[a.get("type", "f32")]
        cnt = int(np.prod(a["domain"]))
        nb = cnt * capi.DTYPE_SIZE[t]
        out[a["name"]] = buf[off:off + nb].view(_NP_DTYPE[t]).reshape(a["domain"])
        off += nb
    return out, bool(coh.value)


def plan(ref_lib: capi.Lib, sc: dict, workers=0, devices=0, oracle_mode=False, suppress=False):
    import ctypes as C

    from paper_2202_05549_b200.api import PlanBuffer
    text = json.dumps(sc).encode()
    nt, npool, na = C.c_int64(0), C.c_int64(0), C.c_int64(0)
    ref_lib.check(ref_lib.scenario_plan(text, workers, devices, int(oracle_mode), int(suppress), None, 0, C.byref(nt), None, 0, C.byref(npool),
                                        None, 0, C.byref(na)))
    tasks = (capi.Task * max(1, nt.value))()
    pool = (C.c_int64 * max(1, npool.value))()
    args = (capi.ArgBinding * max(1, na.value))()
    ref_lib.check(ref_lib.scenario_plan(text, workers, devices, int(oracle_mode), int(suppress), tasks, nt.value, C.byref(nt), pool, npool.value,
                                        C.byref(npool), args, na.value, C.byref(na)))
    return PlanBuffer(tasks[: nt.value], pool, args)
