"""GEMM rasterisation sweep at one size: python scripts/gemm_sweep.py N (env MTB_GEMM_GROUP / MTB_GEMM_NO_PAIR)"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_05549_b200 as mb  # noqa: E402

fn = mb.lib().dll.mt_gemm_bf16_nt
fn.restype = C.c_int
fn.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 6 + [C.c_void_p]
m, n, k = (int(v) for v in sys.argv[1].split("x")) if "x" in sys.argv[1] else (int(sys.argv[1]),) * 3
it = int(sys.argv[2]) if len(sys.argv) > 2 else 3
a = torch.rand(m, k, device="cuda").to(torch.bfloat16)
b = torch.rand(n, k, device="cuda").to(torch.bfloat16)
c = torch.empty(m, n, device="cuda", dtype=torch.float32)
s = torch.cuda.current_stream().cuda_stream
fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, k, k, n, s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(it):
    fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, k, k, n, s)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / it
print(f"mnk={m}x{n}x{k} group={os.environ.get('MTB_GEMM_GROUP', 'default')} nopair={os.environ.get('MTB_GEMM_NO_PAIR', '0')} {ms:.3f} ms {2 * m * n * k / ms / 1e9:.1f} TFLOP/s",
      flush=True)
