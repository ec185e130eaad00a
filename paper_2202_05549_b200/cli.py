"""Command-line front end: `python -m paper_2202_05549_b200 plan|run|fuzz`, the B200 form of the
reference's `manta` tool (proj/tools/manta.cpp:55-180), with the same subcommands, flags,
output lines and exit codes (0 pass, 1 validation / parse / plan error, 2 oracle mismatch or
incoherent replicas, 3 internal error; manta.cpp:15-18, 166-178).

* `plan SCENARIO [--dot FILE]` builds the plan without a GPU and prints per-worker task counts
  by kind (cmd_plan, manta.cpp:55-81); `--dot` writes the task DAG (export_dot, task.cpp:72-110).
* `run SCENARIO [--oracle] [--report FILE]` executes on the GPU(s) (cmd_run, manta.cpp:83-111);
  `--oracle` runs the scenario again in oracle mode (every array on one device, one device)
  on the same executor and compares (compare_results, scenario.cpp:554-603, tolerance 1e-6).
* `fuzz [--cases N] [--seed S]` runs the reference's random scenario campaign
  (run_fuzz_campaign, scenario.cpp:809-846) on the GPU: the scenarios come from the product's
  restatement of make_fuzz_scenario (mt_fuzz_scenario_json), seed for seed the reference's.

System flags follow add_system_flags (manta.cpp:46-54). `--throttle` (default: the scenario's
staging_threshold, 64 MiB) bounds the bytes of chunks in use by issued-but-unfinished tasks per
device like the reference's staging throttle, with its monitor counted in the report
(memory.cpp:290-295, 371-374); `--disk-capacity` sizes the spill file below the pinned-host tier, and
`--seed` randomises the schedule like the reference's seeded ready-task choice
(runtime.cpp:313-319): every task goes to a compute stream drawn from the seeded generator,
behind a random on-device delay (mt_config.schedule_seed); without it tasks run as soon as
their CUDA events allow, concurrently over `--streams` streams per device.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys

import numpy as np

from . import _capi as capi
from . import scenario as S

EXIT_PASS, EXIT_VALIDATION, EXIT_MISMATCH, EXIT_INTERNAL = 0, 1, 2, 3
DEFAULT_DEVICE_CAPACITY = 256 << 20  # system_spec defaults (scenario.hpp:66-73)
DEFAULT_HOST_CAPACITY = 1 << 30
DEFAULT_STAGING_THRESHOLD = 64 << 20  # system_spec::staging_threshold (scenario.hpp:72)
KINDS = ("create", "delete", "execute", "copy", "send", "recv", "reduce")
GOLDEN = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def mix64(h: int) -> int:
    """kernels.cpp:103-110"""
    h &= M64
    h ^= h >> 33
    h = (h * 0xFF51AFD7ED558CCD) & M64
    h ^= h >> 33
    h = (h * 0xC4CEB9FE1A85EC53) & M64
    h ^= h >> 33
    return h


def case_seed(campaign_seed: int, i: int) -> int:
    """run_fuzz_campaign's per-case seed (scenario.cpp:811)"""
    return mix64((campaign_seed + i * GOLDEN) & M64)


def fuzz_scenario(seed: int, lib=None) -> dict:
    """make_fuzz_scenario(seed) as a scenario dict, from the product (mt_fuzz_scenario_json)"""
    from . import lib as product
    lib = lib or product()
    n = C.c_int64(0)
    lib.check(lib.fuzz_scenario_json(seed & M64, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    lib.check(lib.fuzz_scenario_json(seed & M64, buf, n.value + 1, C.byref(n)))
    return json.loads(buf.value)


def load(path: str) -> dict:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise capi.ValidationError(f"cannot open scenario file {path}") from None
    try:
        sc = json.loads(text)
    except json.JSONDecodeError as e:
        raise capi.ValidationError(f"malformed scenario: {e}") from None
    if not isinstance(sc, dict):
        raise capi.ValidationError("malformed scenario: top level must be an object")
    return sc


def system_of(sc: dict, flags) -> dict:
    """the scenario's system block with command-line overrides (to_overrides, manta.cpp:30-44)"""
    s = dict(sc.get("system", {}))
    for key in ("workers", "devices", "device_capacity", "host_capacity", "disk_capacity"):
        v = getattr(flags, key, None) if flags is not None else None
        if v is not None:
            s[key] = v
    if flags is not None and getattr(flags, "throttle", None) is not None:
        s["staging_threshold"] = flags.throttle
    if flags is not None and getattr(flags, "seed", None) is not None and flags.cmd != "fuzz":
        s["ready_seed"] = flags.seed
    s.setdefault("workers", 1)
    s.setdefault("devices", 1)
    if s["workers"] < 1 or s["devices"] < 1:
        raise capi.ValidationError("workers and devices must be at least 1")
    return s


def make_context(sysd: dict, execute: bool, oracle_mode=False, suppress=False, streams=0, compat=False):
    """A context for the scenario's system. Device memory is capped (and the pinned-host spill
    tier enabled) only when the scenario asks for less than the default pool, as the
    reference's memory manager would then evict (memory.cpp:278-376)."""
    from . import context
    workers, devices = (1, 1) if oracle_mode else (sysd["workers"], sysd["devices"])
    cap = int(sysd.get("device_capacity", DEFAULT_DEVICE_CAPACITY))
    spill = execute and not oracle_mode and cap < DEFAULT_DEVICE_CAPACITY
    host = int(sysd.get("host_capacity", DEFAULT_HOST_CAPACITY)) if spill else 0
    disk = int(sysd.get("disk_capacity", 0)) if spill else 0
    return context(workers=workers, devices=devices, execute=execute, num_gpus=1 if execute else 0, suppress_conflict_deps=suppress, compat_deps=compat,
                   streams_per_device=streams, device_capacity=cap if spill else 0, host_capacity=max(host, cap) if spill else 0,
                   staging_threshold=0 if oracle_mode else int(sysd.get("staging_threshold", DEFAULT_STAGING_THRESHOLD)), disk_capacity=disk,
                   schedule_seed=0 if oracle_mode else int(sysd.get("ready_seed", 0) or 0))


def run_scenario(sc: dict, sysd: dict, oracle_mode=False, suppress=False, streams=0, compat=False, trace=False):
    """run_scenario on the GPU: (arrays by name, replicas coherent, report json)"""
    with make_context(sysd, True, oracle_mode, suppress, streams, compat) as ctx:
        if trace:
            ctx.trace(True)
        S.register_gather_kernels(ctx, sc)
        arrays, coherent = S.run(ctx, sc, oracle_mode=oracle_mode)
        report = ctx.report_json()
    return arrays, coherent, report


# -- oracle report (compare_results / oracle_report::to_string, scenario.cpp:554-614) ------
def compare_report(actual: dict, expected: dict, rel_tol=1e-6) -> tuple[bool, str]:
    lines, ok = [], True
    for name, want in expected.items():
        got = actual.get(name)
        same = got is not None and got.shape == want.shape and got.dtype == want.dtype
        max_abs = max_rel = 0.0
        first = -1
        if same:
            g, w = got.ravel(), want.ravel()
            if np.issubdtype(want.dtype, np.integer):
                diff = np.abs(g.astype(np.float64) - w.astype(np.float64))
                bad = np.flatnonzero(g != w)
            else:
                gd, wd = g.astype(np.float64), w.astype(np.float64)
                diff = np.abs(gd - wd)
                den = np.maximum(np.maximum(np.abs(gd), np.abs(wd)), 1e-300)
                rel = np.where(diff == 0, 0.0, diff / den)
                max_rel = float(np.nanmax(rel)) if rel.size else 0.0
                bits = g.view(f"u{g.itemsize}") == w.view(f"u{w.itemsize}")
                bad = np.flatnonzero(~bits & ~(rel <= rel_tol))
            max_abs = float(np.nanmax(diff)) if diff.size else 0.0
            first = int(bad[0]) if bad.size else -1
            same = bad.size == 0
        ok = ok and same
        line = f"  {name}: {'ok' if same else 'MISMATCH'} max_abs={max_abs:g} max_rel={max_rel:g}"
        if first >= 0:
            line += f" first_mismatch={first}"
        lines.append(line)
    return ok, "\n".join(["PASS" if ok else "FAIL"] + lines)


# -- DOT export (export_dot, task.cpp:47-110) ----------------------------------------------
def _box(b) -> str:
    """to_string(rect) (geometry.cpp:96-102): [lo,hi)x[lo,hi)"""
    lo, hi = b
    return "x".join(f"[{a},{c})" for a, c in zip(lo, hi))


_OPS = {0: "+", 1: "*", 2: "min", 3: "max"}


def task_label(t: dict) -> str:
    k = t["kind"]
    s = f"t{t['id']} "
    if k == "create":
        return s + f"Create c{t['chunk']} {_box(t['region'])}"
    if k == "delete":
        return s + f"Delete c{t['chunk']}"
    if k == "execute":
        return s + f"Execute {t['kernel']} {_box(t['sb_blocks'])} @w{t['device'][0]}d{t['device'][1]}"
    if k == "copy":
        return s + f"Copy c{t['src']}->c{t['dst']} {_box(t['dst_region'])}"
    if k == "send":
        return s + f"Send c{t['chunk']} {_box(t['region'])} ->w{t['peer']}"
    if k == "recv":
        return s + f"Recv c{t['chunk']} {_box(t['region'])} <-w{t['peer']}"
    if k == "reduce":
        return s + f"Reduce({_OPS.get(t['op'], '?')}) {len(t['inputs'])} inputs ->c{t['output']}"
    return s + k


def export_dot(tasks: list[dict], workers: int) -> str:
    out = ["digraph plan {", "  rankdir=TB;", "  node [shape=box, fontsize=10];"]
    for w in range(workers):
        out.append(f"  subgraph cluster_worker{w} {{")
        out.append(f'    label="worker {w}";')
        for t in tasks:
            if t["worker"] == w:
                out.append(f'    t{t["id"]} [label="{task_label(t)}"];')
        out.append("  }")
    by_id = sorted(tasks, key=lambda t: t["id"])
    for t in by_id:
        for d in t["deps"]:
            out.append(f"  t{d} -> t{t['id']};")
    sends = {(t["worker"], t["peer"], t["tag"]): t["id"] for t in by_id if t["kind"] == "send"}
    for t in by_id:
        if t["kind"] == "recv":
            s = sends.get((t["peer"], t["worker"], t["tag"]))
            if s is not None:
                out.append(f"  t{s} -> t{t['id']} [style=dashed, constraint=false];")
    out.append("}")
    return "\n".join(out) + "\n"


# -- subcommands ----------------------------------------------------------------------------
def cmd_plan(args) -> int:
    sc = load(args.scenario)
    sysd = system_of(sc, args)
    with make_context(sysd, execute=False, suppress=args.no_conflict_deps, compat=args.compat_deps) as ctx:
        S.register_gather_kernels(ctx, sc)
        S.apply(ctx, sc)
        tasks = ctx.plan()
    launches = sum(int(l.get("repeat", 1)) for l in sc.get("launches", []))
    workers = sysd["workers"]
    for w in range(workers):
        counts: dict = {}
        mine = [t for t in tasks if t["worker"] == w]
        for t in mine:
            counts[t["kind"]] = counts.get(t["kind"], 0) + 1
        print(f"worker {w}:" + "".join(f" {k}={counts[k]}" for k in sorted(counts)) + f" total={len(mine)}")
    print(f"tasks: {len(tasks)} across {workers} workers, {launches} launches")
    if args.dot:
        try:
            with open(args.dot, "w") as f:
                f.write(export_dot(tasks, workers))
        except OSError:
            raise capi.ValidationError(f"cannot write {args.dot}") from None
        print(f"wrote {args.dot}")
    return EXIT_PASS


def _report_totals(report: str) -> dict:
    r = json.loads(report)
    tot = {"evictions": 0, "bytes_sent": 0, "staging_checks": 0, "staging_violations": 0}
    for w in r.get("workers", []):
        for k in tot:
            tot[k] += int(w.get(k, 0))
    return tot


def cmd_run(args) -> int:
    sc = load(args.scenario)
    sysd = system_of(sc, args)
    arrays, coherent, report = run_scenario(sc, sysd, suppress=args.no_conflict_deps, streams=args.streams, compat=args.compat_deps,
                                            trace=bool(args.report))
    t = _report_totals(report)
    print(f"completed: {len(arrays)} arrays, evictions={t['evictions']}, bytes_sent={t['bytes_sent']}, "
          f"staging_checks={t['staging_checks']}, staging_violations={t['staging_violations']}")
    if args.report:
        try:
            with open(args.report, "w") as f:
                f.write(report + "\n")
        except OSError:
            raise capi.ValidationError(f"cannot write {args.report}") from None
        print(f"wrote {args.report}")
    if not coherent:
        print("replica coherence violated: overlapping chunks disagree", file=sys.stderr)
        return EXIT_MISMATCH
    if args.oracle:
        expected, _, _ = run_scenario(sc, sysd, oracle_mode=True)
        ok, text = compare_report(arrays, expected, 1e-6)
        print("oracle: " + text)
        if not ok:
            return EXIT_MISMATCH
    return EXIT_PASS


def cmd_fuzz(args) -> int:
    for i in range(args.cases):
        seed = case_seed(args.seed, i)
        sc = fuzz_scenario(seed)
        try:
            sysd = system_of(sc, None)
            actual, coherent, _ = run_scenario(sc, sysd, suppress=args.no_conflict_deps, streams=args.streams)
            expected, _, _ = run_scenario(sc, sysd, oracle_mode=True)
            ok, text = compare_report(actual, expected, 1e-6)
            message = text if not ok else (None if coherent else "replica coherence violated")
        except capi.MantaError as e:
            message = f"exception: {e}"
        if message:
            print(f"fuzz case {i} (seed {seed}) failed:\n{message}\nscenario:\n{json.dumps(sc, indent=2)}", file=sys.stderr)
            return EXIT_MISMATCH
    print(f"fuzz: {args.cases} cases passed")
    return EXIT_PASS


def _system_flags(p: argparse.ArgumentParser):
    p.add_argument("--workers", type=int, help="Override the scenario's worker count")
    p.add_argument("--devices", type=int, help="Override the devices per worker")
    p.add_argument("--device-capacity", dest="device_capacity", type=int, help="Device memory capacity in bytes")
    p.add_argument("--host-capacity", dest="host_capacity", type=int, help="Host memory capacity in bytes")
    p.add_argument("--disk-capacity", dest="disk_capacity", type=int, help="Disk tier capacity in bytes")
    p.add_argument("--throttle", type=int, help="Staging throttle threshold in bytes")
    p.add_argument("--seed", type=int, help="Randomise the schedule: seeded stream choice and on-device delays per task")
    p.add_argument("--streams", type=int, default=0, help="Compute streams per device (0 = 4)")
    p.add_argument("--no-conflict-deps", dest="no_conflict_deps", action="store_true", help=argparse.SUPPRESS)
    p.add_argument("--compat-deps", dest="compat_deps", action="store_true",
                   help="Whole-chunk dependencies exactly as the reference (default: region-precise)")


def parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="python -m paper_2202_05549_b200",
                                description="B200 runtime with annotation-driven planning (drop-in for the manta tool)")
    sub = p.add_subparsers(dest="cmd", required=True)
    pl = sub.add_parser("plan", help="Build execution plans without running them")
    pl.add_argument("scenario", help="Scenario file")
    pl.add_argument("--dot", default="", help="Write the task DAG in DOT format")
    _system_flags(pl)
    r = sub.add_parser("run", help="Execute a scenario on the GPU(s)")
    r.add_argument("scenario", help="Scenario file")
    r.add_argument("--oracle", action="store_true", help="Compare against the sequential single-device run")
    r.add_argument("--report", default="", help="Write the runtime report as JSON")
    _system_flags(r)
    f = sub.add_parser("fuzz", help="Random scenario campaign checked against the sequential run")
    f.add_argument("--cases", type=int, default=200, help="Number of random scenarios")
    f.add_argument("--seed", type=int, default=1, help="Campaign seed")
    f.add_argument("--streams", type=int, default=0, help="Compute streams per device (0 = 4)")
    f.add_argument("--no-conflict-deps", dest="no_conflict_deps", action="store_true", help=argparse.SUPPRESS)
    return p


def main(argv=None) -> int:
    args = parser().parse_args(argv)
    try:
        if args.cmd == "plan":
            return cmd_plan(args)
        if args.cmd == "run":
            return cmd_run(args)
        return cmd_fuzz(args)
    except (capi.ValidationError, capi.ParseError, capi.PlanError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_VALIDATION
    except Exception as e:  # noqa: BLE001 - the reference maps every other failure to exit 3
        print(f"internal error: {e}", file=sys.stderr)
        return EXIT_INTERNAL
