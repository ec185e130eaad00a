import sys, ctypes as C, torch
sys.path.insert(0, '.')
import paper_2202_05549_b200 as mb
fn = mb.lib().dll.mt_gemm_bf16_nt
fn.restype = C.c_int
fn.argtypes = [C.c_void_p]*3 + [C.c_int64]*6 + [C.c_void_p]
for n in [4096, 8192, 16384, 32768]:
    a = torch.rand(n, n, device='cuda').to(torch.bfloat16)
    b = torch.rand(n, n, device='cuda').to(torch.bfloat16)
    c = torch.empty(n, n, device='cuda', dtype=torch.float32)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(2): fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 10 if n <= 8192 else 3
    e0.record()
    for _ in range(it): fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    ref_ms = None
    if n <= 16384:
        cb = torch.empty(n, n, device='cuda', dtype=torch.bfloat16)
        torch.matmul(a, b.T, out=cb); torch.cuda.synchronize()
        e0.record()
        for _ in range(it): torch.matmul(a, b.T, out=cb)
        e1.record(); torch.cuda.synchronize(); ref_ms = e0.elapsed_time(e1)/it
    print(f"n={n} ours {ms:.3f} ms {2*n**3/ms/1e9:.1f} TFLOP/s  cublas-bf16-out {ref_ms and round(2*n**3/ref_ms/1e9,1)} TFLOP/s", flush=True)
