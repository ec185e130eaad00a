"""The tcgen05 bf16 contraction and cuBLAS (torch.matmul bf16, the MEASURED_PEAKS protocol) at the
same sizes, best of 10 single launches each, interleaved: kernel quality against cuBLAS away from
the power cap that bounds both at 32768^3."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2202_05549_b200 as mb  # noqa: E402

fn = mb.lib().dll.mt_gemm_bf16_nt
fn.restype = C.c_int
fn.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 6 + [C.c_void_p]


def best(call, n, reps=10):
    for _ in range(2):
        call()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        e1.synchronize()
        out.append(2 * n**3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
    return max(out)


res = []
for n in [int(x) for x in (sys.argv[1:] or ["4096", "8192", "16384"])]:
    a = torch.rand(n, n, device="cuda").to(torch.bfloat16)
    b = torch.rand(n, n, device="cuda").to(torch.bfloat16)
    c = torch.empty(n, n, device="cuda", dtype=torch.float32)
    s = torch.cuda.current_stream().cuda_stream
    ours = lambda: fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s)  # noqa: E731
    theirs = lambda: torch.matmul(a, b.T)  # noqa: E731  bf16 output (the MEASURED_PEAKS protocol)
    theirs32 = lambda: torch.mm(a, b.T, out_dtype=torch.float32)  # noqa: E731  f32 output, like ours
    r = {"n": n, "ours": 0.0, "cublas": 0.0, "cublas_f32_out": 0.0}
    for _ in range(3):
        r["ours"] = max(r["ours"], best(ours, n))
        r["cublas"] = max(r["cublas"], best(theirs, n))
        try:
            r["cublas_f32_out"] = max(r["cublas_f32_out"], best(theirs32, n))
        except Exception as e:  # noqa: BLE001
            r["cublas_f32_out"] = str(e)[:80]
    r["ours_over_cublas"] = r["ours"] / r["cublas"]
    if isinstance(r["cublas_f32_out"], float):
        r["ours_over_cublas_f32_out"] = r["ours"] / r["cublas_f32_out"]
    res.append(r)
    del a, b, c
    torch.cuda.empty_cache()
print(json.dumps(res))
