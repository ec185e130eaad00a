import torch, time
for mb in [16, 32, 48, 64, 128, 512]:
    n = mb * (1 << 20) // 4
    a = torch.randn(n, device='cuda'); b = torch.empty_like(a)
    for _ in range(20): b.copy_(a)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    it = 200
    e0.record()
    for _ in range(it): b.copy_(a)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    print(f"{mb} MiB copy: {ms*1e3:.1f} us, {2*mb*(1<<20)/ms/1e9*1e3/1e3:.0f} GB/s")
