"""GPU execution of the reference's own fuzz campaign (make_fuzz_scenario, scenario.cpp:653-849;
acceptance criteria c3/c8): random annotations, distributions and memory caps run through
the B200 planner (region-precise dependencies) and executor (multi-stream, spill tier when
the scenario caps device memory), compared with the reference's sequential oracle run.
Integers (all fuzz arrays are i64) must match bit-exactly and replicas must agree."""
import ctypes as C
import json

import pytest

import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import scenario as S
from oracle import scenario as R

pytestmark = pytest.mark.gpu


def fuzz_scenario(ref, seed):
    n = C.c_int64(0)
    buf = C.create_string_buffer(1 << 20)
    ref.check(ref.fuzz_scenario_json(seed, buf, 1 << 20, C.byref(n)))
    return json.loads(buf.value)


def run_product(sc, suppress=False, streams=0):
    sysd = sc.get("system", {})
    cap = int(sysd.get("device_capacity", 256 << 20))
    spill = cap < (256 << 20)
    with mb.context(workers=sysd.get("workers", 1), devices=sysd.get("devices", 1), num_gpus=1, suppress_conflict_deps=suppress,
                    device_capacity=cap if spill else 0, host_capacity=(1 << 30) if spill else 0, streams_per_device=streams) as ctx:
        S.register_gather_kernels(ctx, sc)
        return S.run(ctx, sc)


def test_correlator_like_scenario(ref, scenarios):
    sc = scenarios["correlator_like"]
    got, coherent = run_product(sc)
    want, _ = R.run(ref, sc, oracle_mode=True)
    assert coherent
    assert S.compare(got, want) == []


@pytest.mark.parametrize("block", range(4))
def test_fuzz_campaign_matches_sequential_oracle(ref, block):
    failures = []
    for i in range(25):
        seed = (0x2545F4914F6CDD1D * (block * 25 + i + 7)) % (1 << 63)
        sc = fuzz_scenario(ref, seed)
        try:
            want, _ = R.run(ref, sc, oracle_mode=True)
        except mb.MantaError:
            continue  # the reference rejects the request sequence too (checked in test_planner_parity)
        got, coherent = run_product(sc)
        problems = S.compare(got, want, 1e-6)
        if problems or not coherent:
            failures.append((seed, problems, coherent))
    assert failures == []


def test_suppressed_conflict_edges_are_detected(ref):
    """Acceptance c8 (mutation power): dropping the conflict edges must break some case. On the
    GPU a dropped edge only shows when the two tasks land on different streams and overlap in
    time, so the campaign uses 16 streams per device and runs until the first detection."""
    broken = tried = 0
    for i in range(160):
        sc = fuzz_scenario(ref, 1000 + i * 7919)
        try:
            want, _ = R.run(ref, sc, oracle_mode=True)
        except mb.MantaError:
            continue
        tried += 1
        try:
            got, coherent = run_product(sc, suppress=True, streams=16)
        except mb.MantaError:
            broken += 1
        else:
            if S.compare(got, want, 1e-6) or not coherent:
                broken += 1
        if broken:
            break
    assert broken > 0, f"no mutation detected in {tried} scenarios"
