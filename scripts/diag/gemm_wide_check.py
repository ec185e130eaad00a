"""Wide CTA-pair tcgen05 kernel (256x512 tiles, MTB_GEMM_WIDE=1) against the single-CTA kernel
(bit-identical expected: same K order per element) and against fp64, on ragged and square
shapes, bf16 and TF32."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2202_05549_b200 as mb  # noqa: E402

lib = mb.lib().dll
for name in ("mt_gemm_bf16_nt", "mt_gemm_tf32_nt"):
    f = getattr(lib, name)
    f.restype = C.c_int
    f.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 6 + [C.c_void_p]


def run(fn, a, b, m, n, k, env):
    for key in ("MTB_GEMM_WIDE", "MTB_GEMM_NO_PAIR", "MTB_GEMM_FORCE_PAIR"):
        os.environ.pop(key, None)
    os.environ.update(env)
    c = torch.full((m, n), float("nan"), device="cuda")
    assert fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, a.stride(0), b.stride(0), n, torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    return c


ok = True
for (m, n, k) in [(4096, 4096, 4096), (2304, 4352, 1024), (4224, 4096 + 256, 512), (8192, 8192, 2048), (3000, 5000, 776), (1024 * 3, 1536, 4096)]:
    for kind in ("bf16", "tf32"):
        if kind == "tf32" and k % 4:
            continue
        g = torch.Generator(device="cuda").manual_seed(m + n + k)
        a = torch.rand(m, k, device="cuda", generator=g) - 0.3
        b = torch.rand(n, k, device="cuda", generator=g) - 0.3
        fn = lib.mt_gemm_bf16_nt if kind == "bf16" else lib.mt_gemm_tf32_nt
        if kind == "bf16":
            a, b = a.to(torch.bfloat16), b.to(torch.bfloat16)
        single = run(fn, a, b, m, n, k, {"MTB_GEMM_NO_PAIR": "1"})
        wide = run(fn, a, b, m, n, k, {"MTB_GEMM_WIDE": "1"})
        ref = (a.double() @ b.double().t())
        err = ((wide.double() - ref).abs().max() / ref.abs().max()).item()
        same = torch.equal(single, wide)
        nan = torch.isnan(wide).any().item()
        print(f"{kind} {m}x{n}x{k}: identical to single-CTA={same} max err/max|C|={err:.2e} nan={nan}", flush=True)
        ok = ok and not nan and err < 1e-3
print("ALL OK" if ok else "FAILED")
