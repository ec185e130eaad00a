#!/bin/bash
# CTA-pair bf16 contraction with the dynamic tile scheduler: rasterisation group (M units) sweep
for n in 32768 16384; do
  for g in 2 4 6 8 16; do
    echo -n "n=$n group=$g: "
    MTB_GEMM_GROUP=$g python - <<PY
import ctypes as C, os, sys, torch
sys.path.insert(0, '.')
import paper_2202_05549_b200 as mb
fn = mb.lib().dll.mt_gemm_bf16_nt; fn.restype = C.c_int; fn.argtypes = [C.c_void_p]*3 + [C.c_int64]*6 + [C.c_void_p]
n = $n
os.environ["MTB_GEMM_FORCE_PAIR"] = "1"
a = torch.rand(n, n, device="cuda").to(torch.bfloat16); b = torch.rand(n, n, device="cuda").to(torch.bfloat16)
c = torch.empty(n, n, device="cuda", dtype=torch.float32); s = torch.cuda.current_stream().cuda_stream
fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s); torch.cuda.synchronize()
best = 0
for _ in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s); e1.record(); e1.synchronize()
    best = max(best, 2 * n**3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
print(f"{best:.1f} TFLOP/s")
PY
  done
done
