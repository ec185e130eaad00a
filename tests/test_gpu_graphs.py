"""CUDA-graph replay of repeated submissions (executor.cu issue_batch / capture / replay): an
iterative heat2d loop over 4 logical devices (execute + halo-copy submissions, period 2) is
captured after its signature repeats and then replayed with one cudaGraphLaunch per launch.
The result must equal, bit for bit, the C oracle and the same loop with replay disabled
(MTB_NO_GRAPHS=1, a fresh process); interleaving a non-replayable launch and host reads must
keep the ordering."""
import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import Arr

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEAT = "global [i, j] => read in[i-1:i+1, j-1:j+1], write out[i,j]"
F32 = C.POINTER(C.c_float)

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import Arr
rows, cols, iters = 512, 768, 25
HEAT = "global [i, j] => read in[i-1:i+1, j-1:j+1], write out[i,j]"
with mb.context(workers=1, devices=4, num_gpus=1) as ctx:
    devs = ctx.devices
    d = lambda: ctx.dist.stencil([rows, cols], [rows // 4, cols], [1, 0], devs)
    a = ctx.create_array([rows, cols], "f32", d(), 0)
    b = ctx.create_array([rows, cols], "f32", d(), 0)
    ctx.write(a, np.random.default_rng(7).standard_normal((rows, cols)).astype(np.float32))
    w = ctx.dist.block_work([rows, cols], [16, 16], [rows // 4, cols], devs)
    for i in range(iters):
        ctx.launch("heat2d", [rows, cols], [16, 16], w, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
        ctx.flush()
        a, b = b, a
        if i == 12:
            mid = ctx.read(a)  # a host read in the middle of the replayed sequence
    out = ctx.read(a)
    st = ctx.exec_stats()
print(json.dumps({"out": out.view(np.uint32).tobytes().hex()[:0], "sum": int(out.view(np.uint32).astype(np.uint64).sum()),
                  "mid": int(mid.view(np.uint32).astype(np.uint64).sum()), "captures": st["graph_captures"], "replays": st["graph_replays"]}))
np.save(sys.argv[2], out)
"""


def _run(tmp_path, env_extra):
    path = tmp_path / "g.py"
    path.write_text(SCRIPT)
    out = tmp_path / f"out_{len(env_extra)}.npy"
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, str(path), ROOT, str(out)], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1]), np.load(out)


def test_replay_matches_unreplayed_and_oracle(tmp_path, okern):
    with_g, out_g = _run(tmp_path, {})
    without, out_n = _run(tmp_path, {"MTB_NO_GRAPHS": "1"})
    assert with_g["captures"] == 2 and with_g["replays"] >= 20  # period-2 pattern: two graphs
    assert without["captures"] == 0 and without["replays"] == 0
    assert np.array_equal(out_g.view(np.uint32), out_n.view(np.uint32))
    assert with_g["mid"] == without["mid"]
    x = np.random.default_rng(7).standard_normal((512, 768)).astype(np.float32)
    cur, nxt = x.copy(), np.empty_like(x)
    for _ in range(25):
        okern.oracle_heat2d(C.c_int64(512), C.c_int64(768), C.c_double(0.1), cur.ctypes.data_as(F32), nxt.ctypes.data_as(F32))
        cur, nxt = nxt, cur
    assert np.array_equal(out_g.view(np.uint32), cur.view(np.uint32))


def test_replay_interleaved_with_other_work(okern):
    """replayed launches, then a launch with different scalars (not replayable as captured),
    then replays again: ordering through the shared completion events"""
    rows, cols = 256, 512
    with mb.context(workers=1, devices=2, num_gpus=1) as ctx:
        devs = ctx.devices
        d = lambda: ctx.dist.stencil([rows, cols], [rows // 2, cols], [1, 0], devs)  # noqa: E731
        a = ctx.create_array([rows, cols], "f32", d(), 0)
        b = ctx.create_array([rows, cols], "f32", d(), 0)
        x = np.random.default_rng(3).standard_normal((rows, cols)).astype(np.float32)
        ctx.write(a, x)
        w = ctx.dist.block_work([rows, cols], [16, 16], [rows // 2, cols], devs)
        alphas = [0.1] * 8 + [0.2] + [0.1] * 8
        for al in alphas:
            ctx.launch("heat2d", [rows, cols], [16, 16], w, [rows, cols, al, Arr(b), Arr(a)], HEAT)
            ctx.flush()
            a, b = b, a
        got = ctx.read(a)
        st = ctx.exec_stats()
    assert st["graph_replays"] > 0
    cur, nxt = x.copy(), np.empty_like(x)
    for al in alphas:
        okern.oracle_heat2d(C.c_int64(rows), C.c_int64(cols), C.c_double(al), cur.ctypes.data_as(F32), nxt.ctypes.data_as(F32))
        cur, nxt = nxt, cur
    assert np.array_equal(got.view(np.uint32), cur.view(np.uint32))


def test_fuzz_scenarios_with_repeats_match_the_reference(ref):
    """the reference's random scenarios with every launch repeated three times: repeated
    submissions are captured and replayed as CUDA graphs (when eligible), and the final arrays
    must still equal the reference's sequential oracle run"""
    import ctypes as C2

    from paper_2202_05549_b200 import scenario as S
    from oracle import scenario as R
    replays = 0
    checked = 0
    for i in range(60):
        seed = (0x9E3779B97F4A7C15 * (i + 101)) % (1 << 64)
        n = C2.c_int64(0)
        buf = C2.create_string_buffer(1 << 20)
        ref.check(ref.fuzz_scenario_json(seed, buf, 1 << 20, C2.byref(n)))
        sc = json.loads(buf.value)
        for launch in sc["launches"]:
            launch["repeat"] = 3
        sc["system"]["device_capacity"] = 256 << 20  # no spill: graphs are eligible
        try:
            want, _ = R.run(ref, sc, oracle_mode=True)
        except mb.MantaError:
            continue
        with mb.context(workers=sc["system"]["workers"], devices=sc["system"]["devices"], num_gpus=1) as ctx:
            S.register_gather_kernels(ctx, sc)
            got, coherent = S.run(ctx, sc)
            replays += ctx.exec_stats()["graph_replays"]
        assert coherent and S.compare(got, want, 1e-6) == [], seed
        checked += 1
    assert checked >= 30 and replays > 0


@pytest.mark.parametrize("per_flush", [4, 10])
def test_multi_launch_submissions_replay_bit_exact(okern, per_flush):
    """several launches handed to the executor in one flush (the bench's C1 pattern): the batch
    is one graph whose edges run across iterations; a trailing partial batch and a batch with a
    second kernel (scale by a different alpha) are replayed or issued eagerly. Bit-exact against
    the oracle either way"""
    rows, cols, iters = 384, 640, 47
    x = np.random.default_rng(per_flush).standard_normal((rows, cols)).astype(np.float32)
    alphas = [0.1 if i % 9 else 0.25 for i in range(iters)]
    with mb.context(workers=1, devices=4, num_gpus=1) as ctx:
        devs = ctx.devices
        d = lambda: ctx.dist.stencil([rows, cols], [rows // 4, cols], [1, 0], devs)  # noqa: E731
        a = ctx.create_array([rows, cols], "f32", d(), 0)
        b = ctx.create_array([rows, cols], "f32", d(), 0)
        ctx.write(a, x)
        w = ctx.dist.block_work([rows, cols], [16, 16], [rows // 4, cols], devs)
        for rep in range(3):  # the same sequence three times: batches repeat and get replayed
            for i, al in enumerate(alphas):
                ctx.launch("heat2d", [rows, cols], [16, 16], w, [rows, cols, al, Arr(b), Arr(a)], HEAT)
                if (i + 1) % per_flush == 0:
                    ctx.flush()
                a, b = b, a
            ctx.flush()
        got = ctx.read(a)
        st = ctx.exec_stats()
    assert st["graph_replays"] > 0
    cur, nxt = x.copy(), np.empty_like(x)
    for _ in range(3):
        for al in alphas:
            okern.oracle_heat2d(C.c_int64(rows), C.c_int64(cols), C.c_double(al), cur.ctypes.data_as(F32), nxt.ctypes.data_as(F32))
            cur, nxt = nxt, cur
    assert np.array_equal(got.view(np.uint32), cur.view(np.uint32))
