#!/usr/bin/env python
"""Event timing of the tcgen05 bf16 contraction at N^3: 2 warm-ups, then 5 launches; prints
best / median TFLOP/s. Kernel choice and schedule follow the MTB_GEMM_* environment."""
import ctypes as C
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_05549_b200 as mb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
pad = int(os.environ.get("GEMM_PAD", "0"))  # extra elements per operand row (row pitch n + pad)
fn = mb.lib().dll.mt_gemm_bf16_nt
fn.restype = C.c_int
fn.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 6 + [C.c_void_p]
a = torch.rand(n, n + pad, device="cuda").to(torch.bfloat16)
b = torch.rand(n, n + pad, device="cuda").to(torch.bfloat16)
c = torch.empty(n, n, device="cuda", dtype=torch.float32)
s = torch.cuda.current_stream().cuda_stream
call = lambda: fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n + pad, n + pad, n, s)  # noqa: E731
for _ in range(2):
    assert call() == 0
torch.cuda.synchronize()
rates = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    call()
    e1.record()
    e1.synchronize()
    rates.append(2 * n**3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
print(f"best {max(rates):.1f} median {statistics.median(rates):.1f} TFLOP/s")
