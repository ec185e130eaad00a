"""Halo copies fused into the producing stencil kernel (executor.cu plan_mirrors, heat2d.cu
mirrors): after a heat2d launch over a row-block stencil distribution the planner emits copy
tasks that move each chunk's boundary rows into its neighbours' halo rows (planner.cpp,
reference planner.cpp:389-517). The executor hands such a copy to the kernel that produces its
source rows, which stores them a second time straight into the neighbour chunk, and the copy
completes with the kernel. Results must equal, bit for bit, the C oracle and the unfused run
(MTB_NO_HALO_FUSION=1), with graph replay on and off, on ragged grids where the kernel cannot
take the mirror (the copy is then issued as usual), and with 3 superblocks per chunk."""
import ctypes as C

import numpy as np
import pytest

import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import Arr, Superblock

pytestmark = pytest.mark.gpu
HEAT = "global [i, j] => read in[i-1:i+1, j-1:j+1], write out[i,j]"
F32 = C.POINTER(C.c_float)


def _oracle(okern, x, iters):
    rows, cols = x.shape
    cur, nxt = x.copy(), np.empty_like(x)
    for _ in range(iters):
        okern.oracle_heat2d(C.c_int64(rows), C.c_int64(cols), C.c_double(0.1), cur.ctypes.data_as(F32), nxt.ctypes.data_as(F32))
        cur, nxt = nxt, cur
    return cur


def _run(rows, cols, parts, iters, strip=0, per_flush=1):
    bj = 16 if cols % 16 == 0 else 2  # block width dividing a ragged row
    x = np.random.default_rng(rows + cols).standard_normal((rows, cols)).astype(np.float32)
    with mb.context(workers=1, devices=parts, num_gpus=1) as ctx:
        devs = ctx.devices
        d = lambda: ctx.dist.stencil([rows, cols], [rows // parts, cols], [1, 0], devs)  # noqa: E731
        a = ctx.create_array([rows, cols], "f32", d(), 0)
        b = ctx.create_array([rows, cols], "f32", d(), 0)
        ctx.write(a, x)
        w = ctx.dist.block_work([rows, cols], [16, bj], [rows // parts, cols], devs)
        if strip:
            rb, sb, cb = rows // parts // 16, strip // 16, (cols + 15) // 16
            w = [Superblock((lo, 0), (hi, cb), dv) for i, dv in enumerate(devs)
                 for lo, hi in ((i * rb, i * rb + sb), (i * rb + sb, (i + 1) * rb - sb), ((i + 1) * rb - sb, (i + 1) * rb))]
        for i in range(iters):
            ctx.launch("heat2d", [rows, cols], [16, bj], w, [rows, cols, 0.1, Arr(b), Arr(a)], HEAT)
            if (i + 1) % per_flush == 0:
                ctx.flush()
            a, b = b, a
        out = ctx.read(a)
        coherent = ctx.replicas_coherent(a)
        st = ctx.exec_stats()
    return x, out, coherent, st


@pytest.mark.parametrize("rows,cols,parts,strip,per_flush", [(512, 768, 4, 0, 1), (512, 768, 4, 0, 5), (1024, 1024, 4, 64, 1),
                                                              (768, 512, 3, 0, 1), (512, 770, 4, 0, 1)])
def test_fused_halo_matches_unfused_and_oracle(okern, monkeypatch, rows, cols, parts, strip, per_flush):
    iters = 20
    x, fused, coh_f, st_f = _run(rows, cols, parts, iters, strip, per_flush)
    monkeypatch.setenv("MTB_NO_HALO_FUSION", "1")
    _, plain, coh_p, st_p = _run(rows, cols, parts, iters, strip, per_flush)
    assert coh_f and coh_p
    assert np.array_equal(fused.view(np.uint32), plain.view(np.uint32))
    assert np.array_equal(fused.view(np.uint32), _oracle(okern, x, iters).view(np.uint32))
    assert st_p["fused_copies"] == 0
    if cols % 4 == 0:
        # every halo row copy after a heat2d launch is stored by its producing kernel: 2 per
        # interior chunk boundary per launch
        assert st_f["fused_copies"] == 2 * (parts - 1) * iters
        assert st_f["copies"] + st_f["fused_copies"] == st_p["copies"]
        assert st_f["bytes_fused"] == 2 * (parts - 1) * iters * cols * 4
    else:  # the kernel's vectorised columns do not cover a ragged row: plain copies
        assert st_f["fused_copies"] == 0 and st_f["copies"] == st_p["copies"]


def test_fused_halo_without_graphs(okern, monkeypatch):
    """with graph replay off (MTB_NO_GRAPHS=1) tasks are issued one at a time without lookahead,
    so nothing is fused and the result is unchanged"""
    monkeypatch.setenv("MTB_NO_GRAPHS", "1")
    x, out, coh, st = _run(512, 768, 4, 10)
    assert coh and st["fused_copies"] == 0
    assert np.array_equal(out.view(np.uint32), _oracle(okern, x, 10).view(np.uint32))
