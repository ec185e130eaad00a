"""Runtime kernel compilation: the user's __device__ kernel with a virtual
block index and manta::Vector/Matrix views, a generated per-instance wrapper with baked
offsets/strides (reference generate_wrapper_source, kernels.cpp:522-596, pinned by
test_kernels.cpp:168-211), compiled by NVRTC for sm_100a. CPU: wrapper text and compile
errors (NVRTC needs no GPU). GPU: the paper's stencil listing runs distributed and matches the
AOT stencil1d bit for bit; a 2D kernel indexes Matrix views with global coordinates."""
import numpy as np
import pytest

import paper_2202_05549_b200 as mb
from paper_2202_05549_b200 import Arr
from paper_2202_05549_b200.api import wrapper_source

STENCIL_PARAMS = [("n", "scalar", "i64", 0, False), ("output", "array", "f32", 1, True), ("input", "array", "f32", 1, False)]
# PAPER.md listing "Modified code" (the user's side of the contract)
STENCIL_SRC = r"""
__device__ void stencil(dim3 virtBlockIdx, int64_t n, manta::Vector<float> output, const manta::Vector<float> input) {
  int64_t i = (int64_t)blockDim.x * virtBlockIdx.x + threadIdx.x;
  if (i >= n) return;
  float left = i - 1 >= 0 ? input[i - 1] : 0;
  float mid = input[i];
  float right = i + 1 < n ? input[i + 1] : 0;
  output[i] = (left + mid + right) / 3.0f;
}
"""


def test_wrapper_reproduces_per_worker_constants(mt):
    src = wrapper_source(mt, "stencil", STENCIL_PARAMS, [1024], [[1024], [1023]], [[1], [1]])
    assert "block_offset_x = 1024" in src
    assert "input_offset_0 = 1023" in src
    assert "output_offset_0 = 1024" in src
    assert 'extern "C" __global__ void stencil_wrapper(' in src
    assert "stencil(virtual_block_index, n, output, input);" in src
    assert "const float *const input_ptr" in src  # read-only stays const


def test_wrapper_two_dimensional_and_deterministic(mt):
    params = [("m", "scalar", "i64", 0, False), ("C", "array", "f32", 2, True), ("A", "array", "f32", 2, False)]
    args = ("mm", params, [4, 0], [[16, 0], [16, 0]], [[64, 1], [64, 1]])
    src = wrapper_source(mt, *args)
    for s in ("C_offset_0 = 16", "C_offset_1 = 0", "C_strides_0 = 64", "C_strides_1 = 1", "block_offset_y = 0"):
        assert s in src
    assert wrapper_source(mt, *args) == src


def test_compile_errors_carry_the_nvrtc_log(mt):
    with mb.context(execute=False) as ctx:
        with pytest.raises(mb.ValidationError, match="does not compile"):
            ctx.compile_kernel("broken", STENCIL_PARAMS, "__device__ void broken(dim3 b, int64_t n, manta::Vector<float> o, const manta::Vector<float> i) { o[0] = undefined_name; }")
        ctx.compile_kernel("stencil", STENCIL_PARAMS, STENCIL_SRC)  # the paper's kernel compiles
        a = ctx.create_array([4096], "f32", ctx.dist.row([4096], 1024, ctx.devices), 1)
        b = ctx.create_array([4096], "f32", ctx.dist.row([4096], 1024, ctx.devices), 0)
        ctx.launch("stencil", [4096], [256], ctx.dist.block_work([4096], [256], [1024], ctx.devices), [4096, Arr(b), Arr(a)],
                   "global i => write output[i], read input[i-1:i+1]")
        assert any(t["kind"] == "execute" for t in ctx.plan())


@pytest.mark.gpu
def test_paper_stencil_matches_aot_stencil1d():
    n, chunk, iters = 100_003, 25_088, 5
    rng = np.random.default_rng(2)
    x0 = rng.standard_normal(n).astype(np.float32)
    ann = "global i => write output[i], read input[i-1:i+1]"
    res = []
    for kernel in ("stencil", "stencil1d"):
        with mb.context(workers=2, devices=2, num_gpus=1) as ctx:
            if kernel == "stencil":
                ctx.compile_kernel("stencil", STENCIL_PARAMS, STENCIL_SRC)
            devs = ctx.devices
            d = lambda: ctx.dist.stencil([n], [chunk], [1], devs)  # noqa: E731
            a, b = ctx.create_array([n], "f32", d(), 0), ctx.create_array([n], "f32", d(), 0)
            ctx.write(a, x0)
            w = ctx.dist.block_work([n], [256], [chunk], devs)
            for _ in range(iters):
                ctx.launch(kernel, [n], [256], w, [n, Arr(b), Arr(a)], ann)
                a, b = b, a
            res.append(ctx.read(a))
    # stencil1d (kernels.cpp:147-165) divides by 3.0f in f32 with the same operation order
    assert np.array_equal(res[0].view(np.uint32), res[1].view(np.uint32))


@pytest.mark.gpu
def test_matrix_views_use_global_indices():
    rows, cols = 640, 384
    params = [("rows", "scalar", "i64", 0, False), ("cols", "scalar", "i64", 0, False), ("out", "array", "f64", 2, True),
              ("in", "array", "f64", 2, False)]
    src = r"""
__device__ void transpose_add(dim3 vb, int64_t rows, int64_t cols, manta::Matrix<double> out, const manta::Matrix<double> in) {
  int64_t i = (int64_t)vb.x * blockDim.x + threadIdx.x, j = (int64_t)vb.y * blockDim.y + threadIdx.y;
  if (i >= rows || j >= cols) return;
  out[i][j] = in(i, j) * 2.0 + (double)(i * 1000 + j);
}
"""
    x = np.random.default_rng(4).standard_normal((rows, cols))
    with mb.context(workers=1, devices=4, num_gpus=1) as ctx:
        ctx.compile_kernel("transpose_add", params, src)
        devs = ctx.devices
        dist = ctx.dist.tile([rows, cols], [rows // 2, cols // 2], devs)
        a, b = ctx.create_array([rows, cols], "f64", dist, 0), ctx.create_array([rows, cols], "f64", ctx.dist.tile([rows, cols], [rows // 2, cols // 2], devs), 0)
        ctx.write(a, x)
        w = ctx.dist.block_work([rows, cols], [16, 16], [rows // 2, cols // 2], devs)
        ctx.launch("transpose_add", [rows, cols], [16, 16], w, [rows, cols, Arr(b), Arr(a)], "global [i, j] => write out[i,j], read in[i,j]")
        got = ctx.read(b)
    i = np.arange(rows)[:, None]
    j = np.arange(cols)[None, :]
    assert np.array_equal(got, x * 2.0 + (i * 1000 + j).astype(np.float64))
