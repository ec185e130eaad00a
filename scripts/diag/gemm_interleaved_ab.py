"""Interleaved A/B of tcgen05 bf16 contraction variants at n^3 under sustained load: `rounds`
rounds, each running every variant for `per` back-to-back launches (device events per launch),
so power-cap clock drift hits all variants alike. Prints per-variant median and best TFLOP/s.
  usage: python scripts/diag/gemm_interleaved_ab.py [n] [rounds] [per] variant...
  variant: single-static | single-dyn-G | pair-static-G | pair-dyn-G | wide-static-G | wide-dyn-G, each
           optionally +rowwise (MTB_GEMM_EPI=0) |
           cublas (torch.mm bf16 -> f32 output, like ours; not compared for bit identity)"""
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
KEYS = ("MTB_GEMM_FORCE_PAIR", "MTB_GEMM_NO_PAIR", "MTB_GEMM_DYNAMIC", "MTB_GEMM_GROUP", "MTB_GEMM_WIDE", "MTB_GEMM_EPI")


def env_of(v):
    if v == "cublas":
        return {}
    rowwise = v.endswith("+rowwise")  # the per-row epilogue stores (MTB_GEMM_EPI=0)
    v = v.removesuffix("+rowwise")
    kind, sched, *g = v.split("-")
    e = {"wide": {"MTB_GEMM_WIDE": "1"}, "pair": {"MTB_GEMM_FORCE_PAIR": "1", "MTB_GEMM_WIDE": "0"},
         "single": {"MTB_GEMM_NO_PAIR": "1"}}[kind]
    if sched == "dyn":
        e["MTB_GEMM_DYNAMIC"] = "1"
    if g:
        e["MTB_GEMM_GROUP"] = g[0]
    if rowwise:
        e["MTB_GEMM_EPI"] = "0"
    return e


tf32 = os.environ.get("GEMM_TF32") == "1"  # f32 operands through mt_gemm_tf32_nt (rounding pass included)
fn = mb.lib().dll.mt_gemm_tf32_nt if tf32 else mb.lib().dll.mt_gemm_bf16_nt
fn.restype = C.c_int
fn.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 6 + [C.c_void_p]
a = torch.rand(n, n, device="cuda")
b = torch.rand(n, n, device="cuda")
if not tf32:
    a, b = a.to(torch.bfloat16), b.to(torch.bfloat16)
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
            if v == "cublas":
                torch.mm(a, b.T, out_dtype=torch.float32)
            else:
                assert fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s) == 0
            e1.record()
            e1.synchronize()
            if r > 0:  # round 0 warms up
                rates[v].append(2.0 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
        if v == "cublas":
            continue
        if ref is None:
            ref = c.clone()
        elif not torch.equal(ref, c):
            print(f"{v}: result differs from {variants[0]}", flush=True)
for v in variants:
    print(f"n={n} {v:14s} median {statistics.median(rates[v]):7.1f} best {max(rates[v]):7.1f} TFLOP/s ({len(rates[v])} launches)", flush=True)
