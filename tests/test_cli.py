"""The command-line front end (`python -m paper_2202_05549_b200 plan|run|fuzz`, the reference's
`manta` tool, proj/tools/manta.cpp) and the product's fuzz-scenario generator
(mt_fuzz_scenario_json, restating make_fuzz_scenario, scenario.cpp:653-807).

CPU: the generator reproduces the reference's scenario for every seed; `plan` prints the
reference's per-worker task counts and, with --compat-deps, writes the reference's DOT byte
for byte; error exit codes. GPU: `run --oracle` over the bundled scenarios and a `fuzz`
campaign end to end."""
import ctypes as C
import json
import os
import subprocess
import sys

import pytest

from paper_2202_05549_b200 import cli
from paper_2202_05549_b200 import scenario as S
from oracle import scenario as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_cli(*args, timeout=600):
    r = subprocess.run([sys.executable, "-m", "paper_2202_05549_b200", *args], capture_output=True, text=True, cwd=ROOT, timeout=timeout)
    return r.returncode, r.stdout, r.stderr


def ref_fuzz(ref, seed):
    n = C.c_int64(0)
    buf = C.create_string_buffer(1 << 20)
    ref.check(ref.fuzz_scenario_json(seed, buf, 1 << 20, C.byref(n)))
    return json.loads(buf.value)


def test_generator_matches_reference_seed_for_seed(mt, ref):
    seeds = [cli.case_seed(1, i) for i in range(200)] + [(i * 0x2545F4914F6CDD1D + 99) % (1 << 64) for i in range(300)] + [0, (1 << 64) - 1]
    for seed in seeds:
        assert cli.fuzz_scenario(seed, mt) == ref_fuzz(ref, seed), seed


def test_mix64_known_values():
    # mix64 is the murmur3 fmix64 finaliser (kernels.cpp:103-110)
    assert cli.mix64(0) == 0
    assert cli.mix64(1) == 0xB456BCFC34C2CB2C
    assert cli.case_seed(1, 0) == cli.mix64(1)


def _write(tmp_path, name, sc):
    p = tmp_path / f"{name}.json"
    p.write_text(json.dumps(sc))
    return str(p)


def _ref_dot(ref, sc):
    text = json.dumps(sc).encode()
    n = C.c_int64(0)
    ref.check(ref.scenario_dot(text, 0, 0, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    ref.check(ref.scenario_dot(text, 0, 0, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


@pytest.mark.parametrize("name", ["compute_only", "correlator_like", "map", "matmul", "nbody_like", "reduction", "spmv", "stencil"])
def test_plan_counts_and_dot_match_reference(ref, scenarios, tmp_path, name):
    sc = scenarios[name]
    path = _write(tmp_path, name, sc)
    dot = str(tmp_path / f"{name}.dot")
    rc, out, err = run_cli("plan", path, "--dot", dot, "--compat-deps")
    assert rc == 0, err
    tasks = R.plan(ref, sc).dicts()
    workers = sc.get("system", {}).get("workers", 1)
    want = []
    for w in range(workers):
        counts = {}
        for t in tasks:
            if t["worker"] == w:
                counts[t["kind"]] = counts.get(t["kind"], 0) + 1
        want.append(f"worker {w}:" + "".join(f" {k}={counts[k]}" for k in sorted(counts)) + f" total={sum(counts.values())}")
    launches = sum(l.get("repeat", 1) for l in sc["launches"])
    want.append(f"tasks: {len(tasks)} across {workers} workers, {launches} launches")
    assert out.splitlines()[:workers + 1] == want
    with open(dot) as f:
        assert f.read() == _ref_dot(ref, sc)
    # region-precise dependencies (the default) change edges, not task counts
    rc, out2, err = run_cli("plan", path)
    assert rc == 0, err
    assert out2.splitlines() == want


def test_exit_codes(tmp_path, scenarios):
    assert run_cli("plan", str(tmp_path / "missing.json"))[0] == cli.EXIT_VALIDATION
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert run_cli("plan", str(bad))[0] == cli.EXIT_VALIDATION
    sc = json.loads(json.dumps(scenarios["stencil"]))
    sc["launches"][0]["annotation"] = "global i => read in[i-1:i+1, write out[i]"  # parse error
    rc, _, err = run_cli("plan", _write(tmp_path, "parse", sc))
    assert rc == cli.EXIT_VALIDATION and "error:" in err
    sc = json.loads(json.dumps(scenarios["stencil"]))
    sc["launches"][0]["kernel"] = "no_such_kernel"
    assert run_cli("plan", _write(tmp_path, "kernel", sc))[0] == cli.EXIT_VALIDATION
    assert run_cli("plan", _write(tmp_path, "ok", scenarios["map"]), "--workers", "0")[0] == cli.EXIT_VALIDATION


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["compute_only", "correlator_like", "map", "matmul", "nbody_like", "reduction", "spmv", "stencil"])
def test_run_oracle_passes(scenarios, tmp_path, name):
    report = str(tmp_path / "report.json")
    rc, out, err = run_cli("run", _write(tmp_path, name, scenarios[name]), "--oracle", "--report", report)
    assert rc == 0, out + err
    assert out.splitlines()[0].startswith("completed: ")
    assert "oracle: PASS" in out
    with open(report) as f:
        r = json.load(f)
    assert len(r["workers"]) == scenarios[name].get("system", {}).get("workers", 1)
    # traced task records like the reference's run_report (runtime.cpp:626-629)
    recs = [t for w in r["workers"] for t in w["tasks"]]
    assert recs and all(0 <= t["start_ns"] <= t["end_ns"] for t in recs)
    kinds = {t["kind"] for t in recs}
    assert "execute" in kinds and kinds <= {"create", "delete", "execute", "copy", "send", "recv", "reduce"}
    if scenarios[name].get("arrays"):
        assert "create" in kinds


@pytest.mark.gpu
def test_fuzz_campaign_passes():
    rc, out, err = run_cli("fuzz", "--cases", "40", "--seed", "1", timeout=1200)
    assert rc == 0, err[-3000:]
    assert out.strip() == "fuzz: 40 cases passed"


@pytest.mark.gpu
def test_run_with_all_memory_tiers(scenarios, tmp_path):
    """`run` with the reference's memory flags small enough that chunks spill to pinned host
    memory and on to the disk tier; still equal to the oracle-mode run"""
    report = str(tmp_path / "report.json")
    rc, out, err = run_cli("run", _write(tmp_path, "stencil", scenarios["stencil"]), "--oracle", "--report", report,
                           "--device-capacity", str(3 * 256_008), "--host-capacity", str(4 * 256_008), "--disk-capacity", str(64 << 20))
    assert rc == 0, out + err
    assert "oracle: PASS" in out
    with open(report) as f:
        r = json.load(f)
    assert sum(w["evictions"] for w in r["workers"]) > 0
    assert sum(w["bytes_host_to_disk"] for w in r["workers"]) > 0
