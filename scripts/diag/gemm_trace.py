"""Per-tile MMA issue times of the CTA-pair bf16 kernel (MTB_GEMM_TRACE, a device buffer address)
at n^3 for the static and dynamic schedules: how far apart in time do tiles sharing an A panel
(same M unit) or a B panel (same N block) run? Prints the spread statistics."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2202_05549_b200 as mb  # noqa: E402

fn = mb.lib().dll.mt_gemm_bf16_nt
fn.restype = C.c_int
fn.argtypes = [C.c_void_p] * 3 + [C.c_int64] * 6 + [C.c_void_p]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
a = torch.rand(n, n, device="cuda").to(torch.bfloat16)
b = torch.rand(n, n, device="cuda").to(torch.bfloat16)
c = torch.empty(n, n, device="cuda", dtype=torch.float32)
units = (n // 256) * (n // 256)
tr = torch.zeros(3 * units, dtype=torch.int64, device="cuda")
group = 16
for variant in ("static", "dynamic"):
    os.environ["MTB_GEMM_FORCE_PAIR"] = "1"
    os.environ.pop("MTB_GEMM_STATIC", None)
    if variant == "static":
        os.environ["MTB_GEMM_STATIC"] = "1"
    os.environ["MTB_GEMM_TRACE"] = str(tr.data_ptr())
    fn(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, n, n, n, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    t = tr.view(units, 3).cpu().numpy().astype(np.int64)
    start = t[:, 1] - t[:, 1].min()
    dur = t[:, 2] - t[:, 1]
    nb_count = n // 256
    ids = np.arange(units)
    g = ids // (group * nb_count)
    r = ids % (group * nb_count)
    mu = g * group + r % group
    nb = r // group
    # spread of start times among tiles sharing a B panel within the same group (16 tiles)
    spreads_b = []
    for key in np.unique(g * nb_count + nb):
        sel = (g * nb_count + nb) == key
        spreads_b.append(start[sel].max() - start[sel].min())
    print(f"{variant}: kernel {(t[:, 2].max() - t[:, 1].min()) / 1e6:.2f} ms, tile median {np.median(dur) / 1e3:.1f} us, "
          f"B-panel start spread median {np.median(spreads_b) / 1e3:.1f} us p90 {np.percentile(spreads_b, 90) / 1e3:.1f} us", flush=True)
    os.environ.pop("MTB_GEMM_TRACE")
