"""One cuBLAS bf16 matmul (torch.matmul, bf16 out) at n^3 with Bt row-major (C = A Bt^T), for ncu."""
import sys

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
a = torch.rand(n, n, device="cuda").to(torch.bfloat16)
bt = torch.rand(n, n, device="cuda").to(torch.bfloat16)
c = torch.matmul(a, bt.t())
torch.cuda.synchronize()
print("ok", n, c.dtype)
