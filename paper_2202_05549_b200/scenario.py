"""Scenario files (the reference's on-disk workload format, proj/src/scenario.cpp:69-181)
driven through the B200 context: the same operation sequence as apply_scenario
(scenario.cpp:394-453) — create arrays, then every launch `repeat` times with optional name
swaps — and the same result gathering (scenario.cpp:471-509) and comparison rule
(compare_results, scenario.cpp:554-603: integers bit-exact, floats bit-equal or within a
relative tolerance).
"""
from __future__ import annotations

import math
from typing import Callable

import numpy as np

from . import _capi as capi
from .api import Arr, Context, ValidationError

_sig_cache: dict = {}


def kernel_signature(ctx: Context, kernel: str) -> list[tuple]:
    """[(name, is_array, dtype, rank, writable)] from the product's kernel registry."""
    key = (ctx.lib.path, kernel)
    if key in _sig_cache:
        return _sig_cache[key]
    import ctypes as C
    n = ctx.lib.kernel_count()
    for i in range(n):
        name = C.create_string_buffer(capi.KERNEL_NAME_MAX)
        params = (capi.ParamSpec * 32)()
        np_ = C.c_int32(0)
        ctx.lib.check(ctx.lib.kernel_info(i, name, capi.KERNEL_NAME_MAX, params, 32, C.byref(np_)))
        sig = [(p.name.decode(), p.kind == capi.PARAM_ARRAY, p.dtype, p.rank, bool(p.writable)) for p in params[: np_.value]]
        _sig_cache[(ctx.lib.path, name.value.decode())] = sig
    if key not in _sig_cache:
        raise ValidationError(f'unknown kernel "{kernel}"')
    return _sig_cache[key]


def make_distribution(ctx: Context, spec: dict, extents: list, devices: list):
    kind = spec["kind"]
    d = ctx.dist
    if kind == "row":
        return d.row(extents, spec["rows"], devices)
    if kind == "col":
        return d.col(extents, spec["cols"], devices)
    if kind == "tile":
        return d.tile(extents, spec["extents"], devices)
    if kind == "stencil":
        return d.stencil(extents, spec["extents"], spec["halo"], devices)
    if kind == "replicated":
        return d.replicated(extents, devices)
    if kind == "single":
        return d.single(extents, devices[0])
    if kind == "custom":
        from .api import Chunk
        return [Chunk(i, tuple(c["lo"]), tuple(c["hi"]), (c["worker"], c["device"])) for i, c in enumerate(spec["chunks"])]
    raise ValidationError(f'unknown distribution kind "{kind}"')


def gather_signature(sc: dict, annotation: str) -> list[tuple]:
    """Signature of the synthesized gather kernel (scenario.cpp:276-286): one array
    parameter per access, in access order; writable when it writes or reduces."""
    from .annotation_text import accesses
    types = {a["name"]: (capi.DTYPE_NAMES[a.get("type", "f32")], len(a["domain"])) for a in sc.get("arrays", [])}
    sig = []
    for name, mode in accesses(annotation):
        if name not in types:
            raise ValidationError(f'gather annotation names unknown array "{name}"')
        t, r = types[name]
        sig.append((name, True, t, r, mode in ("write", "readwrite", "reduce")))
    return sig


def register_gather_kernels(ctx: Context, sc: dict, launcher=None, user_for: Callable | None = None):
    """register_gather_kernels (scenario.cpp:368-389): one context-local `gather@<launch index>`
    kernel per gather launch, with the native GPU body (mt_ctx_gather_register)."""
    import ctypes as C
    arrays = {a["name"]: a for a in sc.get("arrays", [])}
    for index, l in enumerate(sc.get("launches", [])):
        if l["kernel"] != "gather":
            continue
        sig = gather_signature(sc, l["annotation"])
        if launcher is None and ctx.lib.has("ctx_gather_register"):
            n = len(sig)
            types = (C.c_int32 * max(1, n))(*[t for _, _, t, _, _ in sig])
            doms = (capi.Rect * max(1, n))()
            for i, (name, _, _, r, _) in enumerate(sig):
                doms[i] = capi.Rect.make([0] * r, arrays[name]["domain"])
            ctx.lib.check(ctx.lib.ctx_gather_register(ctx.h, f"gather@{index}".encode(), l["annotation"].encode(), n, types, doms))
            _sig_cache[(ctx.lib.path, f"gather@{index}")] = sig
            continue
        params = (capi.ParamSpec * max(1, len(sig)))()
        for i, (name, _, t, r, w) in enumerate(sig):
            params[i].name = name.encode()
            params[i].kind = capi.PARAM_ARRAY
            params[i].dtype = t
            params[i].rank = r
            params[i].writable = int(w)
        user = user_for(sc, l) if user_for else None
        ctx.lib.check(ctx.lib.ctx_kernel_register(ctx.h, f"gather@{index}".encode(), params, len(sig), launcher, user))
        _sig_cache[(ctx.lib.path, f"gather@{index}")] = sig


def apply(ctx: Context, sc: dict, oracle_mode=False, flush=True) -> dict:
    """apply_scenario: returns the final name -> array id map (after swaps)."""
    devices = ctx.devices
    ids: dict = {}
    for a in sc.get("arrays", []):
        ext = list(a["domain"])
        dist = ctx.dist.single(ext, devices[0]) if oracle_mode else make_distribution(ctx, a["distribution"], ext, devices)
        fill = a.get("fill")
        if fill is not None and fill not in (0, 1, 0.0, 1.0):
            raise ValidationError("fill must be 0 or 1")
        if a["name"] in ids:
            raise ValidationError(f'duplicate array name "{a["name"]}"')
        ids[a["name"]] = ctx.create_array(ext, a.get("type", "f32"), dist, None if fill is None else int(fill))
        if flush:
            ctx.flush()
    for index, l in enumerate(sc.get("launches", [])):
        kernel = f"gather@{index}" if l["kernel"] == "gather" else l["kernel"]
        sig = kernel_signature(ctx, kernel)
        if l.get("repeat", 1) < 1:
            raise ValidationError("repeat must be at least 1")
        repeat = l.get("repeat", 1)
        sw = l.get("swap")
        native = repeat > 1 and ctx.lib.has("launch_repeat") and (not sw or (sw[0] in ids and sw[1] in ids))
        for _ in range(1 if native else repeat):
            work = ctx.dist.block_work(l["grid"], l["block"], l["superblock"], devices)
            if len(l.get("args", [])) != len(sig):
                raise ValidationError(f'kernel "{kernel}" takes {len(sig)} arguments')
            args = []
            for spec, (pname, is_array, t, _, _) in zip(l.get("args", []), sig):
                if not is_array:
                    if isinstance(spec, str):
                        raise ValidationError(f'parameter "{pname}" expects a number')
                    if t in (capi.I32, capi.I64):
                        args.append(int(spec) if isinstance(spec, int) else int(math.floor(spec + 0.5) if spec >= 0 else -math.floor(-spec + 0.5)))
                    else:
                        args.append(float(spec))
                else:
                    if not isinstance(spec, str):
                        raise ValidationError(f'parameter "{pname}" expects an array name')
                    if spec not in ids:
                        raise ValidationError(f'unknown array "{spec}"')
                    args.append(Arr(ids[spec]))
            if native:
                # the whole repeat loop in one native call (mt_launch_repeat): same launches, swaps
                # and hand-offs as the loop below
                ctx.launch_repeat(kernel, l["grid"], l["block"], work, args, l["annotation"], repeat,
                                  swap=(ids[sw[0]], ids[sw[1]]) if sw else None, flush_every=1 if flush else -1)
                if sw and repeat % 2:
                    ids[sw[0]], ids[sw[1]] = ids[sw[1]], ids[sw[0]]
                continue
            ctx.launch(kernel, l["grid"], l["block"], work, args, l["annotation"])
            if flush:
                ctx.flush()
            if sw:
                a, b = sw
                if a not in ids or b not in ids:
                    raise ValidationError("swap names an unknown array")
                ids[a], ids[b] = ids[b], ids[a]
    return ids


def run(ctx: Context, sc: dict, oracle_mode=False) -> tuple[dict, bool]:
    """run_scenario: final arrays by name (scenario order) and replica coherence."""
    ids = apply(ctx, sc, oracle_mode)
    ctx.synchronize()
    out = {}
    coherent = True
    for a in sc.get("arrays", []):
        out[a["name"]] = ctx.read(ids[a["name"]])
        coherent = coherent and ctx.replicas_coherent(ids[a["name"]])
    return out, coherent


def compare(actual: dict, expected: dict, rel_tol=1e-6) -> list[str]:
    """compare_results (scenario.cpp:554-603); returns mismatch descriptions."""
    problems = []
    for name, want in expected.items():
        got = actual.get(name)
        if got is None or got.shape != want.shape or got.dtype != want.dtype:
            problems.append(f"{name}: shape/type mismatch")
            continue
        if np.issubdtype(want.dtype, np.integer):
            bad = np.flatnonzero(got.ravel() != want.ravel())
        else:
            g, w = got.ravel().astype(np.float64), want.ravel().astype(np.float64)
            same_bits = got.ravel().view(np.uint8).reshape(-1, got.itemsize).tobytes() == want.ravel().view(np.uint8).reshape(-1, want.itemsize).tobytes()
            if same_bits:
                continue
            err = np.abs(g - w)
            den = np.maximum(np.maximum(np.abs(g), np.abs(w)), 1e-300)
            rel = np.where(err == 0, 0.0, err / den)
            bits_eq = got.ravel().view(f"u{got.itemsize}") == want.ravel().view(f"u{want.itemsize}")
            bad = np.flatnonzero(~bits_eq & ~(rel <= rel_tol))
        if bad.size:
            problems.append(f"{name}: {bad.size} mismatches, first at {bad[0]}")
    return problems
