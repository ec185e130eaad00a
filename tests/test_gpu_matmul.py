"""tcgen05 bf16 contraction (csrc/kernels/matmul_tc.cu) against an fp64 reference of the same
bf16 inputs. Tolerance (north_star: <= 1e-3 for contractions): every element of C within
1e-3 relative of the fp64 result (inputs are non-negative, so there is no cancellation and
the elementwise relative error is meaningful)."""
import ctypes as C

import numpy as np
import pytest

import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import Arr

pytestmark = pytest.mark.gpu
REL = 1e-3


def _gemm_fn():
    fn = mb.lib().dll.mt_gemm_bf16_nt
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p]
    return fn


def pattern(rows, cols, mod, off):
    i = np.arange(rows, dtype=np.int64)[:, None]
    j = np.arange(cols, dtype=np.int64)[None, :]
    return ((i * 31 + j * 17 + off) % mod).astype(np.float32) / mod


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """round-to-nearest-even f32 -> bf16 bit patterns"""
    u = x.astype(np.float32).view(np.uint32)
    r = ((u >> 16) & 1) + 0x7FFF
    return ((u + r) >> 16).astype(np.uint16)


def from_bf16_bits(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


@pytest.mark.parametrize("m,n,k", [(128, 256, 64), (300, 520, 136), (1024, 768, 1000), (2048, 2048, 4096),
                                   # CTA-pair kernel (>= 148 CTAs of 256x256 tiles): odd M-block count, ragged N and K
                                   (4224, 4096, 512), (3000, 4100, 1000)])
def test_gemm_matches_fp64(m, n, k):
    import torch
    a = to_bf16_bits(pattern(m, k, 1000, 7))
    bt = to_bf16_bits(pattern(n, k, 997, 3))
    da = torch.from_numpy(a.view(np.int16)).cuda()
    db = torch.from_numpy(bt.view(np.int16)).cuda()
    dc = torch.full((m, n), float("nan"), dtype=torch.float32, device="cuda")
    rc = _gemm_fn()(da.data_ptr(), db.data_ptr(), dc.data_ptr(), m, n, k, k, k, n, torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    got = dc.cpu().numpy().astype(np.float64)
    want = from_bf16_bits(a).astype(np.float64) @ from_bf16_bits(bt).astype(np.float64).T
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
    assert np.isfinite(got).all()
    assert rel.max() <= REL, rel.max()


def test_matmul_nt_bf16_through_the_planner():
    """C tiled over a 2x2 device grid; A row panels and Bt column panels are assembled into
    per-device temporaries by the planner (replicated-input transfers, planner.cpp:324-347)."""
    m, n, k = 512, 768, 320
    a = to_bf16_bits(pattern(m, k, 1000, 7))
    bt = to_bf16_bits(pattern(n, k, 997, 3))
    with mb.context(workers=2, devices=2, num_gpus=1) as ctx:
        devs = ctx.devices
        A = ctx.create_array([m, k], "bf16", ctx.dist.row([m, k], 128, devs), 0)
        B = ctx.create_array([n, k], "bf16", ctx.dist.row([n, k], 192, devs), 0)
        Cm = ctx.create_array([m, n], "f32", ctx.dist.tile([m, n], [256, 384], devs), 0)
        ctx.write(A, a)
        ctx.write(B, bt)
        work = ctx.dist.block_work([m, n], [16, 16], [256, 384], devs)
        ctx.launch("matmul_nt_bf16", [m, n], [16, 16], work, [m, n, k, Arr(Cm), Arr(A), Arr(B)],
                   "global [i, j] => write C[i,j], read A[i,:], read Bt[j,:]")
        got = ctx.read(Cm).astype(np.float64)
        kinds = [t["kind"] for t in ctx.plan()]
    want = from_bf16_bits(a).astype(np.float64) @ from_bf16_bits(bt).astype(np.float64).T
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
    assert rel.max() <= REL
    assert kinds.count("execute") == 4 and kinds.count("send") > 0


def _tf32_fn():
    fn = mb.lib().dll.mt_gemm_tf32_nt
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p]
    return fn


def tf32_rne(x: np.ndarray) -> np.ndarray:
    """f32 rounded to nearest-even TF32 (10 mantissa bits): the operand values the TF32 path
    multiplies after its rounding pass (matmul_tc.cu tf32_rne)"""
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0xFFF + ((u >> 13) & 1)) & 0xFFFFE000
    return u.astype(np.uint32).view(np.float32)


TF32_REL = 1e-3  # north_star: contractions within 1e-3 (TF32 operands carry 10 mantissa bits)


@pytest.mark.parametrize("m,n,k", [(128, 256, 32), (300, 520, 136), (1024, 768, 1000), (2048, 2048, 4096),
                                   # CTA-pair kernel: odd M-block count, ragged N and K
                                   (4224, 4096, 512), (3000, 4100, 1000)])
def test_gemm_tf32_matches_fp64(m, n, k):
    """the fp32 form of C3 (kind::tf32, f32 accumulation) within 1e-3 of the fp64 product of the
    f32 inputs, without the truncation bias (mean error); and within 1e-4 of the fp64 product of
    the RNE-rounded inputs, which pins the operand conversion (rounding, not the MMA's
    truncation)"""
    import torch
    rng = np.random.default_rng(m + n + k)
    a = pattern(m, k, 1000, 7) if k % 2 else rng.random((m, k), dtype=np.float32)
    bt = pattern(n, k, 997, 3)
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(bt).cuda()
    dc = torch.full((m, n), float("nan"), dtype=torch.float32, device="cuda")
    assert _tf32_fn()(da.data_ptr(), db.data_ptr(), dc.data_ptr(), m, n, k, k, k, n, torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    got = dc.cpu().numpy().astype(np.float64)
    assert np.isfinite(got).all()
    want = a.astype(np.float64) @ bt.astype(np.float64).T
    rel = (got - want) / np.maximum(np.abs(want), 1e-30)
    assert np.abs(rel).max() <= TF32_REL, np.abs(rel).max()
    # no operand-truncation bias (about -2^-11 = -4.9e-4 on this data); what remains is the tensor
    # core's truncating f32 accumulation, about 2^-24 per K=8 step (cuBLAS TF32 shows the same)
    assert abs(rel.mean()) < 2e-5 + (k / 8) * 2.0 ** -23, rel.mean()
    want_r = tf32_rne(a).astype(np.float64) @ tf32_rne(bt).astype(np.float64).T
    rel_r = np.abs(got - want_r) / np.maximum(np.abs(want_r), 1e-30)
    assert rel_r.max() <= 1e-4, (rel_r.max(), np.abs(rel).max())


@pytest.mark.parametrize("n", [4096, 8192])
def test_gemm_tf32_bit_identical_to_cublas(n):
    """on the C3 ramp operands the tcgen05 TF32 contraction equals cuBLAS TF32 (torch.matmul with
    allow_tf32) bit for bit: the residual error against fp64 is the tensor cores' own f32
    accumulation, not this kernel's (profiles/round2/tf32_vs_cublas.json: also all 2^30 elements
    at 32768^3)"""
    import torch
    i = torch.arange(n, dtype=torch.int64, device="cuda")

    def ramp(mod, off):
        return (((i[:, None] * 31 + i[None, :] * 17 + off) % mod).to(torch.float64) / mod).to(torch.float32)

    a, b = ramp(1000, 7), ramp(997, 7)
    ours = torch.empty(n, n, device="cuda", dtype=torch.float32)
    assert _tf32_fn()(a.data_ptr(), b.data_ptr(), ours.data_ptr(), n, n, n, n, n, n, torch.cuda.current_stream().cuda_stream) == 0
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        theirs = a @ b.T
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    torch.cuda.synchronize()
    assert torch.equal(ours.view(torch.int32), theirs.view(torch.int32))


def test_gemm_tf32_nn_reference_layout():
    """mt_gemm_tf32_nn: B row-major K x N (the reference `matmul` layout), transposed and rounded
    in the preparation pass; ragged sizes and a row pitch wider than the matrix"""
    import torch
    fn = mb.lib().dll.mt_gemm_tf32_nn
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p]
    for m, n, k, pad in [(300, 520, 136, 0), (1000, 777, 1001, 3), (2048, 2048, 2048, 0)]:
        a = pattern(m, k, 1000, 7)
        b = np.zeros((k, n + pad), np.float32)
        b[:, :n] = pattern(k, n, 997, 3)
        da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        dc = torch.full((m, n), float("nan"), dtype=torch.float32, device="cuda")
        assert fn(da.data_ptr(), db.data_ptr(), dc.data_ptr(), m, n, k, k, n + pad, n, torch.cuda.current_stream().cuda_stream) == 0
        torch.cuda.synchronize()
        got = dc.cpu().numpy().astype(np.float64)
        want = a.astype(np.float64) @ b[:, :n].astype(np.float64)
        assert (np.abs(got - want) / np.maximum(np.abs(want), 1e-30)).max() <= TF32_REL


def test_reference_matmul_id_runs_on_tensor_cores():
    """the reference's own kernel id `matmul` (kernels.cpp:167-193, B row-major) through the
    planner: a superblock with m*n*k >= 2^30 takes the tcgen05 path (counted launches) and stays
    within 2e-4 of fp64; a small one keeps the scalar kernel, bit-exact to the reference order"""
    lib = mb.lib().dll
    lib.mt_tensor_core_launches.restype = C.c_uint64
    n = 1024
    a, b = pattern(n, n, 1000, 7), pattern(n, n, 997, 3)
    with mb.context(workers=1, devices=2, num_gpus=1) as ctx:
        devs = ctx.devices
        A = ctx.create_array([n, n], "f32", ctx.dist.row([n, n], n // 2, devs), 0)
        B = ctx.create_array([n, n], "f32", ctx.dist.replicated([n, n], devs), 0)
        Cm = ctx.create_array([n, n], "f32", ctx.dist.row([n, n], n // 2, devs), 0)
        ctx.write(A, a)
        ctx.write(B, b)
        before = lib.mt_tensor_core_launches()
        # one superblock of all rows on device 0 (2^30 = m*n*k): the tensor-core path
        work = ctx.dist.block_work([n, n], [16, 16], [n, n], devs[:1])
        ctx.launch("matmul", [n, n], [16, 16], work, [n, n, n, Arr(Cm), Arr(A), Arr(B)], "global [i, j] => write C[i,j], read A[i,:], read B[:,j]")
        got = ctx.read(Cm).astype(np.float64)
        assert lib.mt_tensor_core_launches() == before + 1
        want = a.astype(np.float64) @ b.astype(np.float64)
        assert (np.abs(got - want) / np.abs(want)).max() <= TF32_REL
        # two superblocks of half the rows: below the threshold, the scalar reference-order kernel
        work2 = ctx.dist.block_work([n, n], [16, 16], [n // 2, n], devs)
        ctx.launch("matmul", [n, n], [16, 16], work2, [n, n, n, Arr(Cm), Arr(A), Arr(B)], "global [i, j] => write C[i,j], read A[i,:], read B[:,j]")
        exact = ctx.read(Cm)
        assert lib.mt_tensor_core_launches() == before + 1
    acc = np.zeros((8, n), np.float32)  # reference order for 8 sample rows
    for l in range(n):
        acc = (acc + (a[:8, l:l + 1] * b[l:l + 1, :]).astype(np.float32)).astype(np.float32)
    assert np.array_equal(exact[:8].view(np.uint32), acc.view(np.uint32))


def test_matmul_nt_tf32_through_the_planner():
    m, n, k = 512, 768, 320
    a = pattern(m, k, 1000, 7)
    bt = pattern(n, k, 997, 3)
    with mb.context(workers=1, devices=4, num_gpus=1) as ctx:
        devs = ctx.devices
        A = ctx.create_array([m, k], "f32", ctx.dist.row([m, k], 128, devs), 0)
        B = ctx.create_array([n, k], "f32", ctx.dist.row([n, k], 192, devs), 0)
        Cm = ctx.create_array([m, n], "f32", ctx.dist.tile([m, n], [256, 384], devs), 0)
        ctx.write(A, a)
        ctx.write(B, bt)
        work = ctx.dist.block_work([m, n], [16, 16], [256, 384], devs)
        ctx.launch("matmul_nt_tf32", [m, n], [16, 16], work, [m, n, k, Arr(Cm), Arr(A), Arr(B)],
                   "global [i, j] => write C[i,j], read A[i,:], read Bt[j,:]")
        got = ctx.read(Cm).astype(np.float64)
    want = a.astype(np.float64) @ bt.astype(np.float64).T
    assert (np.abs(got - want) / np.maximum(np.abs(want), 1e-30)).max() <= TF32_REL


@pytest.mark.parametrize("kind", ["bf16", "tf32"])
@pytest.mark.parametrize("m,n,k", [(4096, 4096, 1024), (4224, 4352, 512), (3000, 5000, 776), (2304, 9472, 256)])
def test_wide_pair_kernel_matches_single_cta(kind, m, n, k, monkeypatch):
    """the wide CTA-pair kernel (256x512 tiles, two M256 N256 MMAs per K step into the 512 TMEM
    columns; the default for M*N > 16384^2 with K > 16384, forced here with MTB_GEMM_WIDE=1 at
    test sizes, dynamic tile counter included) gives bit-identical C to the single-CTA kernel
    (same K order per element) on ragged M / N / K and odd 512-column unit counts, within 1e-3
    of fp64"""
    import torch
    rng = np.random.default_rng(m * 7 + n + k)
    a = rng.random((m, k), dtype=np.float32)
    bt = rng.random((n, k), dtype=np.float32)
    if kind == "bf16":
        a, bt = from_bf16_bits(to_bf16_bits(a)), from_bf16_bits(to_bf16_bits(bt))
        da = torch.from_numpy(to_bf16_bits(a).view(np.int16)).cuda()
        db = torch.from_numpy(to_bf16_bits(bt).view(np.int16)).cuda()
        fn = _gemm_fn()
    else:
        da, db = torch.from_numpy(a).cuda(), torch.from_numpy(bt).cuda()
        fn = _tf32_fn()

    def run(env):
        for key in ("MTB_GEMM_WIDE", "MTB_GEMM_NO_PAIR", "MTB_GEMM_FORCE_PAIR"):
            monkeypatch.delenv(key, raising=False)
        for key, v in env.items():
            monkeypatch.setenv(key, v)
        dc = torch.full((m, n), float("nan"), dtype=torch.float32, device="cuda")
        assert fn(da.data_ptr(), db.data_ptr(), dc.data_ptr(), m, n, k, k, k, n, torch.cuda.current_stream().cuda_stream) == 0
        torch.cuda.synchronize()
        return dc

    mb.lib().dll.mt_tensor_core_launches.restype = C.c_uint64
    before = mb.lib().dll.mt_tensor_core_launches()
    wide = run({"MTB_GEMM_WIDE": "1"})
    single = run({"MTB_GEMM_NO_PAIR": "1"})
    assert mb.lib().dll.mt_tensor_core_launches() >= before + 2
    assert torch.isfinite(wide).all()
    assert torch.equal(wide, single)
    got = wide.cpu().numpy().astype(np.float64)
    want = a.astype(np.float64) @ bt.astype(np.float64).T
    assert (np.abs(got - want) / np.abs(want)).max() <= 1e-3
