"""Interleaved A/B of tcgen05 bf16 contraction variants at n^3 under sustained load: `rounds`
rounds, each running every variant for `per` back-to-back launches (device events per launch),
so power-cap clock drift hits all variants alike. Prints per-variant median and best TFLOP/s.
  usage: python scripts/diag/gemm_interleaved_ab.py [n] [rounds] [per] variant...
  variant: single-static | single-dyn-G | pair-static-G | pair-dyn-G"""
import ctypes as C
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2202_05549_b200 as mb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 8
per = int(sys.argv[3]) if len(sys.argv) > 3 else 3
variants = sys.argv[4:] or ["single-static", "pair-dyn-4"]
KEYS = ("MTB_GEMM_FORCE_PAIR", "MTB_GEMM_NO_PAIR", "MTB_GEMM_DYNAMIC", "MTB_GEMM_GROUP")


def env_of(v):
    kind, sched, *g = v.split("-")
    e = {"MTB_GEMM_FORCE_PAIR" if kind == "pair" else "MTB_GEMM_NO_PAIR": "1"}
    if sched == "dyn":
        e["MTB_GEMM_DYNAMIC"] = "1"
    if g:
        e["MTB_GEMM_GROUP"] = g[0]
    return e


fn = mb.lib().dll.mt_gemm_bf16_nt
fn.restype = C.c_int
fn.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 6 + [C.c_void_p]
a = torch.rand(n, n, device="cuda").to(torch.bfloat16)
b = torch.rand(n, n, device="cuda").to(torch.bfloat16)
c = torch.empty(n, n, device="cuda", dtype=torch.float32)
s = torch.cuda.current_stream().cuda_stream
rates = {v: [] for v in variants}
ref = None
for r in range(rounds + 1):
    for v in variants:
        for k in KEYS:
            os.environ.pop(k, None)
        os.environ.update(env_of(v))
        for _ in range(per):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assert fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s) == 0
            e1.record()
            e1.synchronize()
            if r > 0:  # round 0 warms up
                rates[v].append(2.0 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
        if ref is None:
            ref = c.clone()
        elif not torch.equal(ref, c):
            print(f"{v}: result differs from {variants[0]}", flush=True)
for v in variants:
    print(f"n={n} {v:14s} median {statistics.median(rates[v]):7.1f} best {max(rates[v]):7.1f} TFLOP/s ({len(rates[v])} launches)", flush=True)
