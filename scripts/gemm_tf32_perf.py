#!/usr/bin/env python
"""kind::tf32 contraction throughput (C3 fp32 form): C = A x Bt^T, f32 operands, at the given
size (default 16384^3), CUDA-event timed after warm-up; rel. error vs fp64 on a sampled block."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_05549_b200 as mb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
fn = mb.lib().dll.mt_gemm_tf32_nt
fn.restype = C.c_int
fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p]
i = torch.arange(n, device="cuda", dtype=torch.int64)[:, None]
j = torch.arange(n, device="cuda", dtype=torch.int64)[None, :]
a = ((i * 31 + j * 17 + 7) % 1000).float() / 1000
bt = ((i * 31 + j * 17 + 3) % 997).float() / 997
c = torch.empty(n, n, device="cuda", dtype=torch.float32)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    assert fn(a.data_ptr(), bt.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s) == 0
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    fn(a.data_ptr(), bt.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
ref = a[:256].double() @ bt[:256].double().T
rel = ((c[:256, :256].double() - ref).abs() / ref.abs().clamp_min(1e-30)).max().item()
tf = 2.0 * n ** 3 / (ms / 1e3) / 1e12
print(json.dumps({"n": n, "ms": ms, "tflops": tf, "max_rel_err_vs_fp64": rel}))
