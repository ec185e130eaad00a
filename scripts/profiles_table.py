"""Regenerate the bench-line table at the top of profiles/round2/README.md from
profiles/round2/bench_full.json and bench_reference_arm.json."""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles", "round2")
d = json.loads(open(os.path.join(P, "bench_full.json")).read().strip().splitlines()[-1])
r = json.loads(open(os.path.join(P, "bench_reference_arm.json")).read().strip().splitlines()[-1])
c, h, k = d["contraction"], d["reductions"]["histogram"], d["reductions"]["kmeans"]
sg = d["small_grid"]["roofline"]
rows = [
    ("heat2d 65536² (headline `value`)", f"{d['value'] / 1e9:.0f} Gcell/s",
     f"{d['roofline']['frac']:.2f} of the {d['roofline']['peak']:.0f} GB/s measured copy peak (SM median {d['clocks']['sm_mhz']:.0f} MHz, {', '.join(d['clocks']['reasons']) or 'no throttle'}); DRAM traffic 1.014× algorithmic (`heat2d_tma_ncu_summary.json`)"),
    ("heat2d e2e (host buffers, pipelined, public API)", f"{d['e2e']['value'] / 1e9:.0f} Gcell/s",
     f"synchronous {d['e2e']['sequential']['value'] / 1e9:.0f}; 16 GiB up + 16 GiB down per 100-iteration step"),
    ("reference CPU executor (`--impl reference`)", f"{r['value'] / 1e6:.0f} Mcell/s", f"{r['cpu_baseline']['cores']} host threads"),
    ("C3 contraction 32768³ bf16 (tcgen05 wide CTA pairs)", f"{c['value']:.0f} TFLOP/s",
     f"{c['roofline']['frac']:.2f} of the {c['roofline']['peak']:.0f} burst cuBLAS figure, {c['roofline']['frac_of_sustained']:.2f} of sustained, "
     f"{c['roofline']['frac_of_cublas_same_size']:.2f} of cuBLAS at the same size"),
    ("C3 fp32 operands as TF32", f"{c['tf32']['value']:.0f} TFLOP/s",
     f"{c['tf32']['roofline']['frac']:.2f} of measured cuBLAS TF32; bit-identical to cuBLAS TF32 on every element (`tf32_vs_cublas.json`)"),
    ("C4 histogram 4e9 → 256 bins", f"{h[0]['value'] / 1e12:.2f} T elements/s", f"{h[0]['roofline']['frac']:.2f} of the copy peak (read-only stream)"),
    ("C4 histogram 4e9 → 65536 bins", f"{h[1]['value'] / 1e12:.2f} T elements/s",
     f"{h[1]['roofline']['frac']:.2f} (branch-free common path, `ncu/histogram65536_summary.txt`)"),
    ("C4 k-means assign 1e9×16, k=256", f"{k['assign']['ms']:.0f} ms",
     f"{k['assign']['roofline']['frac']:.2f} of nominal FFMA, {k['assign']['roofline']['frac_of_measured_ffma']:.2f} of the measured FFMA ceiling (`ffma2_probe.txt`)"),
    ("C4 k-means update", f"{k['update']['ms']:.1f} ms", f"{k['update']['roofline']['frac']:.2f} of the copy peak"),
    ("C1 heat 4096², 4 chunks", f"{d['small_grid']['value'] / 1e9:.0f} Gcell/s",
     f"{sg['frac']:.2f} of the HBM line, {sg.get('frac_of_same_size_copy') or float('nan'):.2f} of a same-size device copy"),
    ("n-body n=65536 f64", f"{d['nbody']['value'] / 1e9:.0f} G pairs/s", f"{d['nbody']['roofline']['frac']:.2f} of the FP64 pipe (`ncu/nbody_summary.txt`)"),
    ("C5 out-of-core heat (80 GiB, 24 GiB device cap)", f"{d['out_of_core']['s_per_iter']:.2f} s/iteration",
     f"{d['out_of_core']['time_over_bound']:.2f}× the duplex pinned-link bound (target ≤ 1.5)"),
]
table = "| Leg | Value | Against |\n|---|---|---|\n" + "".join(f"| {a} | {b} | {cc} |\n" for a, b, cc in rows)
readme = os.path.join(P, "README.md")
s = open(readme).read()
s = re.sub(r"\| Leg \| Value \| Against \|\n\|---\|---\|---\|\n(\|.*\|\n)+", table, s, count=1)
open(readme, "w").write(s)
print(table)
