"""The reference's planning acceptance criteria that need no GPU
(proj/tests/acceptance/acceptance.cpp), run against this planner.

* c1 (acceptance.cpp:82-102): interval evaluation of access regions equals per-thread
  enumeration on 1000 random (annotation, superblock, block size, domains) cases. The cases
  follow make_random_region_case (tests/support/oracles.hpp:131-330: 1-3 axes, global / block /
  local bindings, one binding space per expression, single indices, full / one-sided / centred
  two-sided slices kept non-empty per thread) with Python's own RNG; the brute force is
  brute_force_regions (oracles.hpp:24-117) restated in numpy: every thread of the superblock
  evaluates every index, the bounding box of the per-thread boxes is clipped to the domain. Our
  side is the region the planner records for that superblock's execute task (mt_plan_accesses),
  through a launch of a synthesized gather kernel over a work list whose middle superblock is
  the random one.
* c2 (acceptance.cpp:104-156): the three reference annotations parse to their exact trees
  (restated below), and the parsed trees equal the reference parser's (mt_annotation_describe vs
  the shim's mr_annotation_describe over the same canonical rendering) on the c1 annotations,
  every annotation of the bundled scenarios and 100 fuzz scenarios, and malformed texts (same
  error class).
* c6 (acceptance.cpp:247-287): a halo-1 stencil on 2 workers x 2 devices with 4 superblocks moves
  exactly 4 copies and 2 send/recv pairs per iteration and creates no temporaries (both
  dependency modes).
"""
import ctypes as C
import itertools
import random

import numpy as np
import pytest

import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import Arr
from paper_2202_05549_b200 import _capi as capi
from paper_2202_05549_b200.api import Superblock, dtype_code

VARS = ["i", "j", "k"]
BLOCK_VARS = ["bi", "bj", "bk"]
LOCAL_VARS = ["li", "lj", "lk"]


def _random_case(rng: random.Random):
    pick = rng.randint
    rank = pick(1, 3)
    block = [pick(1, 4) for _ in range(rank)]
    grid = [pick(2, 512 if rank == 1 else 40 if rank == 2 else 12) for _ in range(rank)]
    sb_lo, sb_hi = [], []
    for k in range(rank):
        blocks = -(-grid[k] // block[k])
        b0 = pick(0, blocks - 1)
        b1 = pick(b0 + 1, blocks)
        sb_lo.append(b0 * block[k])
        sb_hi.append(b1 * block[k])
    use_block, use_local = pick(0, 2) == 0, pick(0, 2) == 0

    def names(v):
        return v[0] if rank == 1 else "[" + ", ".join(v[:rank]) + "]"

    text = "global " + names(VARS)
    spaces = [VARS[:rank]]
    if use_block:
        text += ", block " + names(BLOCK_VARS)
        spaces.append(BLOCK_VARS[:rank])
    if use_local:
        text += ", local " + names(LOCAL_VARS)
        spaces.append(LOCAL_VARS[:rank])
    ranges = {}
    for k in range(rank):
        ranges[VARS[k]] = (sb_lo[k], sb_hi[k] - 1)
        ranges[BLOCK_VARS[k]] = (sb_lo[k] // block[k], (sb_hi[k] - 1) // block[k])
        ranges[LOCAL_VARS[k]] = (0, block[k] - 1)

    def random_expr():
        pool = spaces[pick(0, len(spaces) - 1)]
        terms = [(pool[pick(0, len(pool) - 1)], pick(-3, 3)) for _ in range(pick(1, 2))]
        return terms, pick(-5, 5)

    def expr_text(e):
        terms, const = e
        out = ""
        for n, (var, c) in enumerate(terms):
            out += ("+" if c >= 0 and n else "") + f"{c}*{var}"
        return out + ("+" if const >= 0 else "") + str(const)

    def range_of(e):
        terms, const = e
        folded = {}
        for var, c in terms:
            folded[var] = folded.get(var, 0) + c
        lo = hi = const
        for var, c in folded.items():
            a, b = c * ranges[var][0], c * ranges[var][1]
            lo, hi = lo + min(a, b), hi + max(a, b)
        return lo, hi

    domains, accesses = [], []
    for a in range(pick(1, 3)):
        arank = pick(1, 3)
        ext = [pick(4, 512 if arank == 1 else 32) for _ in range(arank)]
        domains.append(ext)
        idx = []
        for k in range(arank):
            kind = pick(0, 4)
            if kind == 0:
                idx.append(expr_text(random_expr()))
            elif kind == 1:
                idx.append(":")
            elif kind in (2, 3):
                e = None
                for _ in range(20):
                    cand = random_expr()
                    lo, hi = range_of(cand)
                    if (kind == 2 and hi <= ext[k] - 1) or (kind == 3 and lo >= 0):
                        e = cand
                        break
                idx.append(":" if e is None else (expr_text(e) + ":" if kind == 2 else ":" + expr_text(e)))
            else:
                center = expr_text(random_expr())
                idx.append(f"{center}-{pick(0, 3)}:{center}+{pick(0, 3)}")
        accesses.append("read " + "ABC"[a] + "[" + ",".join(idx) + "]")
    return text + " => " + ", ".join(accesses), grid, block, (sb_lo, sb_hi), domains


def _eval_linear(expr: str, env: dict) -> np.ndarray:
    """value of a generated linear expression ('2*i+-1*bj+3') for every thread"""
    expr = expr.replace("+-", "-")
    total = 0
    for tok in expr.replace("-", "+-").split("+"):
        if not tok:
            continue
        if "*" in tok:
            c, var = tok.split("*")
            total = total + int(c) * env[var]
        else:
            total = total + int(tok)
    return np.broadcast_to(np.asarray(total, dtype=np.int64), env["i"].shape)


def _brute_force(text, block, sb, domains):
    """brute_force_regions (oracles.hpp:24-117): per-thread boxes, their bounding box, clipped"""
    rank = len(block)
    axes = [np.arange(sb[0][k], sb[1][k], dtype=np.int64) for k in range(rank)]
    g = np.meshgrid(*axes, indexing="ij")
    env = {}
    for k in range(rank):
        env[VARS[k]] = g[k].ravel()
        env[BLOCK_VARS[k]] = g[k].ravel() // block[k]
        env[LOCAL_VARS[k]] = g[k].ravel() % block[k]
    out = []
    for acc, dom in zip(text.split("=>")[1].split("read ")[1:], domains):
        idx = acc.strip().rstrip(",").strip()[2:-1].split(",")
        n = env["i"].shape[0]
        alive = np.ones(n, bool)
        los, his = [], []
        for k, ix in enumerate(idx):
            if ":" in ix:
                lo_t, hi_t = ix.split(":")
                lo = _eval_linear(lo_t, env) if lo_t else np.zeros(n, np.int64)
                hi = _eval_linear(hi_t, env) if hi_t else np.full(n, dom[k] - 1, np.int64)
            else:
                lo = hi = _eval_linear(ix, env)
            alive &= lo <= hi
            los.append(lo)
            his.append(hi)
        if not alive.any():
            out.append(None)
            continue
        lo = [max(0, int(x[alive].min())) for x in los]
        hi = [min(dom[k], int(x[alive].max()) + 1) for k, x in enumerate(his)]
        out.append(None if any(a >= b for a, b in zip(lo, hi)) else (tuple(lo), tuple(hi)))
    return out


def _planned_regions(text, grid, block, sb, domains):
    ctx = mb.context(workers=1, devices=1, execute=False, record_accesses=True)
    dev = ctx.devices[0]
    n = len(domains)
    types = (C.c_int32 * n)(*([dtype_code("f32")] * n))
    doms = (capi.Rect * n)()
    for a, ext in enumerate(domains):
        doms[a] = capi.Rect.make([0] * len(ext), ext)
    ctx.lib.check(ctx.lib.ctx_gather_register(ctx.h, b"region_case", text.encode(), n, types, doms))
    arrays = [ctx.create_array(ext, "f32", ctx.dist.single(ext, dev), 0) for ext in domains]
    # a work list covering the block grid whose middle superblock is the random one
    rank = len(block)
    nblocks = [-(-grid[k] // block[k]) for k in range(rank)]
    cuts = [sorted({0, sb[0][k] // block[k], sb[1][k] // block[k], nblocks[k]}) for k in range(rank)]
    work, target = [], None
    for cell in itertools.product(*[range(len(c) - 1) for c in cuts]):
        lo = tuple(cuts[k][cell[k]] for k in range(rank))
        hi = tuple(cuts[k][cell[k] + 1] for k in range(rank))
        if lo == tuple(sb[0][k] // block[k] for k in range(rank)):
            target = len(work)
        work.append(Superblock(lo, hi, dev))
    first, last = ctx.launch("region_case", grid, block, work, [Arr(x) for x in arrays], text)
    execs = [t["id"] for t in ctx.plan(first, last) if t["kind"] == "execute"]
    task = execs[target]
    chunk_of = {ctx.chunks(x)[0].id: a for a, x in enumerate(arrays)}
    got = [None] * n
    for t, chunk, (lo, hi), _ in ctx.accesses():
        if t == task:
            got[chunk_of[chunk]] = (tuple(lo), tuple(hi))
    ctx.close()
    return got


def test_c1_region_evaluation_equals_enumeration():
    rng = random.Random(20240801)
    failures = []
    for case in range(1000):
        text, grid, block, sb, domains = _random_case(rng)
        want = _brute_force(text, block, sb, domains)
        got = _planned_regions(text, grid, block, sb, domains)
        if got != want:
            failures.append((case, text, sb, got, want))
    assert not failures, failures[:5]


@pytest.mark.parametrize("compat", [True, False])
def test_c6_halo_stencil_transfers_per_iteration(compat):
    ctx = mb.context(workers=2, devices=2, execute=False, compat_deps=compat)
    n = 256000
    devs = ctx.devices
    a = ctx.create_array([n], "f32", ctx.dist.stencil([n], [64000], [1], devs), 1)
    b = ctx.create_array([n], "f32", ctx.dist.stencil([n], [64000], [1], devs), 0)
    work = ctx.dist.block_work([n], [16], [64000], devs)
    assert len(work) == 4
    for _ in range(4):
        first, last = ctx.launch("stencil1d", [n], [16], work, [n, Arr(b), Arr(a)], "global i => read input[i-1:i+1], write output[i]")
        kinds = [t["kind"] for t in ctx.plan(first, last)]
        assert (kinds.count("copy"), kinds.count("send"), kinds.count("recv"), kinds.count("create")) == (4, 2, 2, 0)
        for t in ctx.plan(first, last):
            if t["kind"] == "copy":
                assert not ctx.chunk_meta(t["src"])[2] and not ctx.chunk_meta(t["dst"])[2]
        a, b = b, a
    ctx.close()


def _describe(lib, text):
    buf = C.create_string_buffer(1 << 16)
    n = C.c_int64(0)
    lib.check(lib.annotation_describe(text.encode(), buf, len(buf), C.byref(n)))
    return buf.value.decode()


def _e(const=0, **terms):
    return [const, [[v, c] for v, c in terms.items()]]


def test_c2_reference_annotations_parse_to_exact_trees():
    import json
    i, j = _e(i=1), _e(j=1)
    cases = {
        "global i => read A[i-1:i+1], write B[i]": {
            "bindings": [["global", ["i"]]],
            "accesses": [["A", "read", "+", [["slice", _e(-1, i=1), _e(1, i=1)]]], ["B", "write", "+", [["single", i]]]]},
        "global [i, j] => read A[i,:], read B[:,j], write C[i,j]": {
            "bindings": [["global", ["i", "j"]]],
            "accesses": [["A", "read", "+", [["single", i], ["slice", None, None]]], ["B", "read", "+", [["slice", None, None], ["single", j]]],
                         ["C", "write", "+", [["single", i], ["single", j]]]]},
        "global [i, j] => read A[i,j], reduce(+) sum[i]": {
            "bindings": [["global", ["i", "j"]]],
            "accesses": [["A", "read", "+", [["single", i], ["single", j]]], ["sum", "reduce", "+", [["single", i]]]]},
    }
    lib = mb.lib()
    for text, tree in cases.items():
        assert json.loads(_describe(lib, text)) == tree, text


def test_annotation_trees_match_reference_parser(ref):
    import json
    import os
    lib = mb.lib()
    texts = []
    rng = random.Random(20240801)
    texts += [_random_case(rng)[0] for _ in range(1000)]
    scen = os.path.join(os.path.dirname(__file__), "..", "paper_2202_05549_b200", "scenarios")
    gold = os.path.join(os.path.dirname(__file__), "golden")
    for d in (scen, gold):
        if os.path.isdir(d):
            for f in sorted(os.listdir(d)):
                if f.endswith(".json"):
                    try:
                        sc = json.load(open(os.path.join(d, f)))
                    except ValueError:
                        continue
                    for one in ([sc] if isinstance(sc, dict) and "launches" in sc else sc.values() if isinstance(sc, dict) else []):
                        if isinstance(one, dict):
                            texts += [l["annotation"] for l in one.get("launches", []) if isinstance(l, dict) and "annotation" in l]
    n = C.c_int64(0)
    buf = C.create_string_buffer(1 << 20)
    for seed in range(1, 101):
        ref.check(ref.fuzz_scenario_json(seed * 0x9E3779B97F4A7C15 % (1 << 63), buf, len(buf), C.byref(n)))
        texts += [l["annotation"] for l in json.loads(buf.value)["launches"]]
    texts += ["global [i, j] => read A[i*j]", "global i => read A[i", "global i => frob A[i]", "global i, global i => read A[i]",
              "global i => read A[2*i+3*i-5*i]", "global [i, j] => readwrite A[-i+-j:]", "global i => reduce(min) m[0], reduce(*) p[i:i]",
              "block b, local l => write X[4*b+l]", "global i =>", "=> read A[i]", "global i => read A[k]", "global i => read A[i, ]"]
    assert len(texts) > 1100
    errors = 0
    for text in texts:
        got = want = None
        try:
            got = _describe(lib, text)
        except mb.MantaError as e:
            got = type(e).__name__
        try:
            want = _describe(ref, text)
        except mb.MantaError as e:
            want = type(e).__name__
        assert got == want, text
        errors += got.endswith("Error")
    assert 8 <= errors <= 20, errors  # the malformed texts fail in both parsers, the rest parse
