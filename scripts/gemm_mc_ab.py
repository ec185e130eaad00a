#!/usr/bin/env python
"""A/B of the 32768^3 contraction on the single-CTA kernel with and without the Bt multicast
across a CTA pair (MTB_GEMM_MC), alternated in one process (device events, 3 launches each)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_05549_b200 as mb  # noqa: E402

fn = mb.lib().dll.mt_gemm_bf16_nt
fn.restype = C.c_int
fn.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 6 + [C.c_void_p]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
a = torch.rand(n, n, device="cuda").to(torch.bfloat16)
b = torch.rand(n, n, device="cuda").to(torch.bfloat16)
c = torch.empty(n, n, device="cuda", dtype=torch.float32)
s = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ref = None
for r in range(4):
    for mcv in ("1", "0"):
        os.environ["MTB_GEMM_MC"] = mcv
        assert fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s) == 0
        torch.cuda.synchronize()
        if r == 0:
            sample = c[:: n // 64, :: n // 64].clone()
            if ref is None:
                ref = sample
            else:
                print("max |diff| between variants:", float((sample - ref).abs().max()))
        e0.record()
        for _ in range(3):
            fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print("mc" if mcv == "1" else "plain", round(ms, 2), "ms", round(2 * n ** 3 / ms / 1e9, 1), "TFLOP/s", flush=True)
