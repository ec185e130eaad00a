"""Accuracy of cuBLAS (torch.matmul) on the C3 operands at n^3, next to an fp64 product: the
tensor cores' own f32 accumulation error floor (bias from truncating accumulation), to compare
with the tcgen05 kernels' check in bench.py (full_check)."""
import json
import sys

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
dev = torch.device("cuda")


def ramp(mod, off, kind):
    i = torch.arange(n, dtype=torch.int64, device=dev)
    v = (((i[:, None] * 31 + i[None, :] * 17 + off) % mod).to(torch.float64) / mod).to(torch.float32)
    return v.to(torch.bfloat16) if kind == "bf16" else v


out = {}
for kind in ("bf16", "tf32"):
    a, b = ramp(1000, 7, kind), ramp(997, 7, kind)
    want = a.to(torch.float64) @ b.to(torch.float64).T
    torch.backends.cuda.matmul.allow_tf32 = kind == "tf32"
    got = (a @ b.T).to(torch.float64)
    rel = (got - want) / want.abs()
    out[kind] = {"max_rel": float(rel.abs().max()), "mean_rel": float(rel.mean())}
    del a, b, want, got, rel
    torch.cuda.empty_cache()
print(json.dumps({"n": n, "cublas": out}))
