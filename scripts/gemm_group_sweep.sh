#!/bin/bash
# single-CTA tcgen05 GEMM at 32768^3: rasterisation group sweep (device-event timing)
for g in 16 32 64 12 24; do
  MTB_GEMM_GROUP=$g python - <<PY
import ctypes as C, torch, sys
sys.path.insert(0, '.')
import paper_2202_05549_b200 as mb
fn = mb.lib().dll.mt_gemm_bf16_nt
fn.restype = C.c_int
fn.argtypes = [C.c_void_p]*3 + [C.c_int64]*6 + [C.c_void_p]
n = 32768
a = torch.rand(n, n, device='cuda').to(torch.bfloat16); b = torch.rand(n, n, device='cuda').to(torch.bfloat16)
c = torch.empty(n, n, device='cuda', dtype=torch.float32); s = torch.cuda.current_stream().cuda_stream
fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3): fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s)
e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / 3
print("group $g", round(ms, 2), "ms", round(2 * n**3 / ms / 1e9, 1), "TFLOP/s")
PY
done
