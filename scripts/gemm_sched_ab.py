"""A/B of the tcgen05 bf16 contraction's tile scheduling (matmul_tc.cu): the CTA-pair kernel with
the static round robin (MTB_GEMM_STATIC=1) vs the dynamic counter, and the single-CTA kernel
(MTB_GEMM_NO_PAIR=1), at n^3; device events, best of `reps` launches; results checked equal
across variants (same tiles, same K order per tile)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_05549_b200 as mb  # noqa: E402

fn = mb.lib().dll.mt_gemm_bf16_nt
fn.restype = C.c_int
fn.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 6 + [C.c_void_p]
VARIANTS = {"pair-static": {"MTB_GEMM_FORCE_PAIR": "1", "MTB_GEMM_STATIC": "1"}, "pair-dynamic": {"MTB_GEMM_FORCE_PAIR": "1"},
            "pair-dyn-g8": {"MTB_GEMM_FORCE_PAIR": "1", "MTB_GEMM_GROUP": "8"},
            "single-static": {"MTB_GEMM_NO_PAIR": "1", "MTB_GEMM_STATIC": "1"}, "single-dynamic": {"MTB_GEMM_NO_PAIR": "1"},
            "single-dyn-g8": {"MTB_GEMM_NO_PAIR": "1", "MTB_GEMM_GROUP": "8"}, "default": {}}
sizes = [int(x) for x in sys.argv[1:]] or [8192, 16384, 32768]
for n in sizes:
    a = torch.rand(n, n, device="cuda").to(torch.bfloat16)
    b = torch.rand(n, n, device="cuda").to(torch.bfloat16)
    ref = None
    for name, env in VARIANTS.items():
        for k in ("MTB_GEMM_FORCE_PAIR", "MTB_GEMM_STATIC", "MTB_GEMM_NO_PAIR", "MTB_GEMM_GROUP"):
            os.environ.pop(k, None)
        os.environ.update(env)
        c = torch.empty(n, n, device="cuda", dtype=torch.float32)
        s = torch.cuda.current_stream().cuda_stream
        assert fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s) == 0
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(3 if n >= 32768 else 6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s)
            e1.record()
            e1.synchronize()
            best = max(best, 2.0 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
        same = None
        if True:
            if ref is None:
                ref = c.clone()
            else:
                same = bool(torch.equal(ref, c))
        print(f"n={n} {name:13s} {best:7.1f} TFLOP/s" + ("" if same is None else f" identical-to-first={same}"), flush=True)
        del c
    del a, b, ref
    torch.cuda.empty_cache()
