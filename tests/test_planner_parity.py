"""Plan parity with the reference driver (proj/src/planner.cpp) — SURVEY Appendix B item 10.

* compat_deps mode: the task sequence is IDENTICAL to the reference's (ids, kinds,
  workers/resources, chunk ids and regions, fills, argument bindings, copy regions, tags,
  reduce input order AND dependency lists), checked against the committed golden plans and
  against the live reference on the bundled scenarios and on the reference's own fuzz
  generator (make_fuzz_scenario, scenario.cpp:653-812), including which requests fail.
* region mode (the default): the same tasks with region-precise dependency lists whose
  transitive closure (a) is contained in the reference's and (b) still orders every pair of
  conflicting accesses (overlapping regions of one chunk, at least one write): the
  serial-order guarantee the reference pins in test_array_registry.cpp:102-149.
"""
import ctypes as C
import json
import os

import pytest

import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import Arr
from paper_2202_05549_b200 import scenario as S
from oracle import scenario as R

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def product_plan(sc, compat, oracle_mode=False, record=False):
    w = 1 if oracle_mode else sc.get("system", {}).get("workers", 1)
    d = 1 if oracle_mode else sc.get("system", {}).get("devices", 1)
    ctx = mb.context(workers=w, devices=d, execute=False, compat_deps=compat, record_accesses=record)
    S.register_gather_kernels(ctx, sc)
    S.apply(ctx, sc, oracle_mode=oracle_mode, flush=False)
    return ctx


def normalize(plan):
    # JSON round trip turns tuples into lists
    return json.loads(json.dumps(plan))


def strip_deps(plan):
    return [{k: v for k, v in t.items() if k != "deps"} for t in plan]


def closure(plan):
    """task id -> set of transitive predecessors"""
    reach = {}
    for t in plan:
        s = set()
        for d in t["deps"]:
            s.add(d)
            s |= reach[d]
        reach[t["id"]] = s
    return reach


def assert_orders_conflicts(ctx, plan):
    reach = closure(plan)
    by_chunk = {}
    for task, chunk, (lo, hi), write in ctx.accesses():
        by_chunk.setdefault(chunk, []).append((task, lo, hi, write))
    for chunk, recs in by_chunk.items():
        for i in range(len(recs)):
            ta, la, ha, wa = recs[i]
            for j in range(i + 1, len(recs)):
                tb, lb, hb, wb = recs[j]
                if ta == tb or not (wa or wb):
                    continue
                if any(max(x0, y0) >= min(x1, y1) for x0, x1, y0, y1 in zip(la, ha, lb, hb)):
                    continue  # disjoint regions: no ordering needed
                assert ta in reach[tb], f"chunk {chunk}: task {tb} not ordered after conflicting task {ta}"


@pytest.mark.parametrize("name", ["compute_only", "correlator_like", "map", "matmul", "nbody_like", "reduction", "spmv", "stencil"])
@pytest.mark.parametrize("mode", ["system", "oracle"])
def test_bundled_scenarios_compat_plans_match_golden(name, mode, scenarios):
    with open(os.path.join(GOLDEN, "plans.json")) as f:
        gold = json.load(f)[name][mode]
    ctx = product_plan(scenarios[name], compat=True, oracle_mode=(mode == "oracle"))
    assert normalize(ctx.plan()) == gold


@pytest.mark.parametrize("name", ["compute_only", "correlator_like", "map", "matmul", "nbody_like", "reduction", "spmv", "stencil"])
def test_bundled_scenarios_region_plans(name, scenarios):
    with open(os.path.join(GOLDEN, "plans.json")) as f:
        gold = json.load(f)[name]["system"]
    ctx = product_plan(scenarios[name], compat=False, record=True)
    plan = normalize(ctx.plan())
    assert strip_deps(plan) == strip_deps(gold)
    mine, theirs = closure(plan), closure(gold)
    for t in plan:
        assert mine[t["id"]] <= theirs[t["id"]], t["id"]
    assert_orders_conflicts(ctx, plan)


def fuzz_scenario(ref, seed):
    n = C.c_int64(0)
    buf = C.create_string_buffer(1 << 20)
    ref.check(ref.fuzz_scenario_json(seed, buf, 1 << 20, C.byref(n)))
    return json.loads(buf.value)


@pytest.mark.parametrize("block", range(4))
def test_fuzz_plans_match_reference(ref, block):
    for i in range(50):
        seed = 0x9E3779B97F4A7C15 * (block * 50 + i + 1) % (1 << 63)
        sc = fuzz_scenario(ref, seed)
        try:
            want, want_err = normalize(R.plan(ref, sc).dicts()), None
        except mb.MantaError as e:
            want, want_err = None, type(e)
        try:
            ctx = product_plan(sc, compat=True)
            got, got_err = normalize(ctx.plan()), None
        except mb.MantaError as e:
            got, got_err = None, type(e)
        assert got_err == want_err, seed
        if want is None:
            continue
        assert got == want, seed
        # region mode on the same request sequence
        rctx = product_plan(sc, compat=False, record=True)
        rplan = normalize(rctx.plan())
        assert strip_deps(rplan) == strip_deps(want), seed
        theirs = closure(want)
        for t, r in closure(rplan).items():
            assert r <= theirs[t], (seed, t)
        assert_orders_conflicts(rctx, rplan)


def test_region_mode_unchains_halo_stencil():
    """SURVEY finding 3: with whole-chunk tracking every execute of a halo stencil launch
    waits for its left neighbour; region-precise tracking leaves the executes of one launch
    mutually independent."""
    def executes(compat):
        ctx = mb.context(workers=1, devices=4, execute=False, compat_deps=compat)
        n = 4096
        dev = ctx.devices
        a = ctx.create_array([n], "f32", ctx.dist.stencil([n], [1024], [1], dev), 1)
        b = ctx.create_array([n], "f32", ctx.dist.stencil([n], [1024], [1], dev), 0)
        w = ctx.dist.block_work([n], [16], [1024], dev)
        f, l = ctx.launch("stencil1d", [n], [16], w, [n, Arr(b), Arr(a)], "global i => read input[i-1:i+1], write output[i]")
        plan = ctx.plan()
        reach = closure(plan)
        ex = [t["id"] for t in plan if t["kind"] == "execute" and f <= t["id"] < l]
        return sum(1 for x in ex for y in ex if x < y and x in reach[y])
    assert executes(compat=True) == 6  # serial chain of 4 executes
    assert executes(compat=False) == 0


ERROR_CASES = [
    ("stencil1d", "global i => read input[i-1:i+1], write output[i*i]"),  # nonlinear
    ("stencil1d", "global i => read input[i-1:i+1], write output[j]"),  # unbound
    ("stencil1d", "global i => read input[i-1:i+1], write input[i]"),  # duplicate argument
    ("stencil1d", "global i => read input[i-1:i+1]"),  # parameter not annotated
    ("stencil1d", "global i => read input[i-1:i+1], write output[i], read extra[i]"),  # not a parameter
    ("stencil1d", "global i => read input[i-1:i+1], write output[0]"),  # overlapping writes
    ("stencil1d", "global i => read input[i-1:i+1], write output[i, i]"),  # rank mismatch
    ("stencil1d", "global [i, j] => read input[i-1:i+1], write output[i]"),  # too many variables
    ("stencil1d", "global i => read input[i-1:i+1], write output[2*3]"),  # constant product
    ("stencil1d", "global i => read input[i-1:i+1], write output[i] extra"),  # trailing tokens
    ("nokernel", "global i => read input[i], write output[i]"),  # unknown kernel
]


@pytest.mark.parametrize("kernel,ann", ERROR_CASES)
def test_error_kinds_match_reference(ref, kernel, ann):
    import oracle

    def attempt(ctx):
        n = 256
        dev = ctx.devices
        a = ctx.create_array([n], "f32", ctx.dist.stencil([n], [64], [1], dev), 1)
        b = ctx.create_array([n], "f32", ctx.dist.stencil([n], [64], [1], dev), 0)
        w = ctx.dist.block_work([n], [16], [64], dev)
        try:
            ctx.launch(kernel, [n], [16], w, [n, Arr(b), Arr(a)], ann)
        except mb.MantaError as e:
            msg = str(e)
            return type(e).__name__, msg[: msg.index(":", 16)] if isinstance(e, mb.ParseError) else None
        return None, None

    got = attempt(mb.context(workers=2, devices=2, execute=False))
    want = attempt(oracle.reference_context(workers=2, devices=2, execute=False))
    assert got == want
    assert got[0] is not None


def test_read_before_fill_is_a_plan_error(ref):
    import oracle
    for ctx in (mb.context(execute=False), oracle.reference_context(execute=False)):
        n = 64
        a = ctx.create_array([n], "f32", ctx.dist.single([n], (0, 0)))  # fill none
        b = ctx.create_array([n], "f32", ctx.dist.single([n], (0, 0)), 0)
        w = ctx.dist.block_work([n], [16], [64], ctx.devices)
        with pytest.raises(mb.PlanError):
            ctx.launch("stencil1d", [n], [16], w, [n, Arr(b), Arr(a)], "global i => read input[i-1:i+1], write output[i]")


def test_planning_cost_is_subquadratic():
    """the reference needs 40.8 ms per 512-superblock heat launch (O(S^2)
    checks); the indexed planner stays in the low milliseconds."""
    import time
    n = 65536
    ctx = mb.context(workers=1, devices=8, execute=False)
    dev = ctx.devices
    a = ctx.create_array([n, n], "f32", ctx.dist.stencil([n, n], [128, n], [1, 0], dev), 1)
    b = ctx.create_array([n, n], "f32", ctx.dist.stencil([n, n], [128, n], [1, 0], dev), 0)
    w = ctx.dist.block_work([n, n], [16, 16], [128, n], dev)
    assert len(w) == 512
    t0 = time.perf_counter()
    for _ in range(3):
        ctx.launch("heat2d", [n, n], [16, 16], w, [n, n, 0.1, Arr(b), Arr(a)], "global [i, j] => read in[i-1:i+1, j-1:j+1], write out[i,j]")
        a, b = b, a
    per_launch_ms = (time.perf_counter() - t0) / 3 * 1e3
    assert per_launch_ms < 20.0, per_launch_ms
