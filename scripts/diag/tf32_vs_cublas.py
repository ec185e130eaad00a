"""The tcgen05 TF32 contraction (mt_gemm_tf32_nt: RNE-rounded operands, kind::tf32) against
cuBLAS TF32 (torch.matmul, allow_tf32) and an fp64 product on the C3 ramp operands: element-wise
bit identity with cuBLAS and both error statistics (the tensor cores' f32 accumulation floor)."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2202_05549_b200 as mb  # noqa: E402

dev = torch.device("cuda")
fn = mb.lib().dll.mt_gemm_tf32_nt
fn.restype = C.c_int
fn.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 6 + [C.c_void_p]


def ramp(n, mod, off):
    i = torch.arange(n, dtype=torch.int64, device=dev)
    return (((i[:, None] * 31 + i[None, :] * 17 + off) % mod).to(torch.float64) / mod).to(torch.float32)


res = []
for n in [int(x) for x in (sys.argv[1:] or ["8192", "32768"])]:
    a, b = ramp(n, 1000, 7), ramp(n, 997, 7)
    ours = torch.empty(n, n, device=dev, dtype=torch.float32)
    assert fn(a.data_ptr(), b.data_ptr(), ours.data_ptr(), n, n, n, n, n, n, torch.cuda.current_stream().cuda_stream) == 0
    torch.backends.cuda.matmul.allow_tf32 = True
    theirs = a @ b.T
    torch.cuda.synchronize()
    same = int((ours.view(torch.int32) == theirs.view(torch.int32)).sum())
    want = a.to(torch.float64) @ b.to(torch.float64).T
    r = {"n": n, "elements": n * n, "bit_identical_to_cublas": same}
    for name, got in (("ours", ours), ("cublas", theirs)):
        rel = (got.to(torch.float64) - want) / want.abs()
        r[name] = {"max_rel": float(rel.abs().max()), "mean_rel": float(rel.mean())}
        del rel
    res.append(r)
    del a, b, ours, theirs, want
    torch.cuda.empty_cache()
print(json.dumps(res))
