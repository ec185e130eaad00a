#!/usr/bin/env python
"""A/B of the 32768^3 contraction: one launch (single-CTA kernel) vs 16384^2 blocks of C on the
CTA-pair kernel, alternated in one process (device-event timing, 3 launches per sample)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2202_05549_b200 as mb  # noqa: E402

fn = mb.lib().dll.mt_gemm_bf16_nt
fn.restype = C.c_int
fn.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 6 + [C.c_void_p]
n = 32768
a = torch.rand(n, n, device="cuda").to(torch.bfloat16)
b = torch.rand(n, n, device="cuda").to(torch.bfloat16)
c = torch.empty(n, n, device="cuda", dtype=torch.float32)
s = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(4):
    for split in (True, False):
        if split:
            os.environ.pop("MTB_GEMM_NO_SPLIT", None)
        else:
            os.environ["MTB_GEMM_NO_SPLIT"] = "1"
        fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s)
        e0.record()
        for _ in range(3):
            fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print("split" if split else "whole", round(ms, 2), "ms", round(2 * n ** 3 / ms / 1e9, 1), "TFLOP/s", flush=True)
