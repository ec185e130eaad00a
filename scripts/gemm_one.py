#!/usr/bin/env python
"""One tcgen05 GEMM launch of size N^3 (bf16 in, f32 out) for ncu captures."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_05549_b200 as mb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
pad = int(os.environ.get("GEMM_PAD", "0"))  # extra elements per operand row (row pitch n + pad)
fn = mb.lib().dll.mt_gemm_bf16_nt
fn.restype = C.c_int
fn.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 6 + [C.c_void_p]
a = torch.rand(n, n + pad, device="cuda").to(torch.bfloat16)
b = torch.rand(n, n + pad, device="cuda").to(torch.bfloat16)
c = torch.empty(n, n, device="cuda", dtype=torch.float32)
s = torch.cuda.current_stream().cuda_stream
assert fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n + pad, n + pad, n, s) == 0
torch.cuda.synchronize()
print("ok", n)
