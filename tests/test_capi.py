"""The C-ABI library loads without a GPU and exports every symbol include/manta_b200.h
declares; the oracle shim exports the same entry points with the mr_ prefix."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    with open(os.path.join(ROOT, "include", "manta_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(mt_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ["mt_ctx_create", "mt_array_create", "mt_launch", "mt_sync", "mt_exec_submit", "mt_exec_sync", "mt_exec_read_chunk",
                 "mt_kernel_register", "mt_dist_tile", "mt_work_block", "mt_plan_export", "mt_last_error"]:
        assert must in names


def test_product_exports_every_declared_symbol(mt):
    missing = [n for n in declared() if not hasattr(mt.dll, n)]
    assert missing == []


def test_reference_shim_exports_the_same_entry_points(ref):
    optional = {"mt_exec_stats", "mt_exec_last_stream", "mt_kernel_info", "mt_ctx_kernel_register", "mt_exec_mark", "mt_exec_elapsed_ms",
                "mt_exec_profile", "mt_exec_kernel_time", "mt_exec_trace", "mt_plan_accesses", "mt_ctx_gather_register", "mt_ctx_peer_export",
                "mt_ctx_peer_import", "mt_ctx_nccl_unique_id", "mt_ctx_nccl_init", "mt_array_write_async", "mt_array_read_async", "mt_array_write_box_async", "mt_array_read_box_async", "mt_ctx_kernel_compile", "mt_wrapper_source",
                "mt_gemm_bf16_nt", "mt_gemm_tf32_nt", "mt_gemm_tf32_nn", "mt_tensor_core_launches", "mt_plan_cache_hits"}  # GPU-only: the reference has no tensor-core contraction
    missing = [n for n in declared() if n not in optional and not hasattr(ref.dll, "mr_" + n[3:])]
    assert missing == []


def test_version_and_kernel_registry(mt):
    assert b"sm_100a" in mt.version()
    assert mt.kernel_count() >= 25


def test_plan_only_context_needs_no_gpu(mt):
    import paper_2202_05549_b200 as mb
    with mb.context(workers=2, devices=2, execute=False) as ctx:
        assert ctx.devices == [(0, 0), (0, 1), (1, 0), (1, 1)]
        a = ctx.create_array([64], "f32", ctx.dist.row([64], 16, ctx.devices), 1)
        assert [c.id for c in ctx.chunks(a)] == [0, 1, 2, 3]
        assert ctx.plan_size() == 4


def test_errors_map_to_reference_kinds(mt):
    import paper_2202_05549_b200 as mb
    with mb.context(execute=False) as ctx:
        a = ctx.create_array([16], "f32", ctx.dist.single([16], (0, 0)), 1)
        w = ctx.dist.block_work([16], [4], [16], ctx.devices)
        with pytest.raises(mb.PlanError):
            ctx.launch("no_such_kernel", [16], [4], w, [], "global i =>")
        with pytest.raises(mb.ParseError):
            ctx.launch("fill", [16], [4], w, [16, 1.0, mb.Arr(a)], "global i => write out[i*i]")
        with pytest.raises(mb.ValidationError):
            ctx.launch("fill", [16], [4], w, [16, 1, mb.Arr(a)], "global i => write out[i]")


def test_executing_context_fails_loudly_without_gpu(mt):
    import paper_2202_05549_b200 as mb
    from conftest import HAS_GPU
    if HAS_GPU:
        pytest.skip("a GPU is present")
    with pytest.raises(mb.ExecutionError):
        mb.context(execute=True)
