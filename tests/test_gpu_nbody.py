"""nbody_like (kernels.cpp:369-401) at sizes past the bundled scenario: the shared-memory tiled
kernel keeps the reference's ascending-j accumulation with IEEE-rounded f64 operations, so it
matches a numpy restatement of the same loop bit for bit (numpy elementwise ops are single
IEEE operations, no contraction)."""
import numpy as np
import pytest

import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import Arr

pytestmark = pytest.mark.gpu


def nbody_ref(pos):
    n, d = pos.shape
    acc = np.zeros((n, d))
    idx = np.arange(n)
    for j in range(n):
        diff = pos[j][None, :] - pos  # (pos_j - pos_i) per i
        dist2 = np.full(n, 1e-3)
        for q in range(d):
            dist2 = dist2 + diff[:, q] * diff[:, q]
        inv = 1.0 / (dist2 * np.sqrt(dist2))
        upd = diff * inv[:, None]
        mask = idx != j
        acc[mask] = acc[mask] + upd[mask]
    return acc


@pytest.mark.parametrize("n,d", [(2000, 3), (777, 2), (300, 1)])
def test_nbody_tiled_bit_exact(n, d):
    rng = np.random.default_rng(n)
    pos = rng.standard_normal((n, d))
    with mb.context(workers=1, devices=2, num_gpus=1) as ctx:
        devs = ctx.devices
        p = ctx.create_array([n, d], "f64", ctx.dist.replicated([n, d], devs), 0)
        half = -(-n // 2)
        f = ctx.create_array([n, d], "f64", ctx.dist.row([n, d], half, devs), 0)
        ctx.write(p, pos)
        sb = -(-half // 64) * 64
        ctx.launch("nbody_like", [n], [64], ctx.dist.block_work([n], [64], [sb], devs), [n, d, Arr(f), Arr(p)],
                   "global i => write force[i,:], read pos[:,:]")
        got = ctx.read(f)
    want = nbody_ref(pos)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_nbody_tiled_slow_paths_bit_exact():
    """magnitudes that push dist2 * sqrt(dist2) past 2^1021 (reciprocal slow path, subnormal
    result) and dist2 to infinity (square-root slow path): the branch-free groups fall back to
    the intrinsics and stay bit-identical to the IEEE loop"""
    n, d = 1000, 3
    rng = np.random.default_rng(7)
    scale = 10.0 ** rng.choice([0.0, 100.0, 102.0, 102.5, 103.0, 150.0, 160.0], size=(n, 1))
    pos = rng.standard_normal((n, d)) * scale
    with mb.context(workers=1, devices=1, num_gpus=1) as ctx:
        dv = ctx.devices
        p = ctx.create_array([n, d], "f64", ctx.dist.single([n, d], dv[0]), 0)
        f = ctx.create_array([n, d], "f64", ctx.dist.single([n, d], dv[0]), 0)
        ctx.write(p, pos)
        ctx.launch("nbody_like", [n], [64], ctx.dist.block_work([n], [64], [-(-n // 64) * 64], dv), [n, d, Arr(f), Arr(p)],
                   "global i => write force[i,:], read pos[:,:]")
        got = ctx.read(f)
    with np.errstate(over="ignore", invalid="ignore"):
        want = nbody_ref(pos)
    assert not np.isnan(want).any()
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
