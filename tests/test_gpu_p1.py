"""GPU tests of the P1 device runtime (include/wgpf_device.cuh): the buffers
it flushes are KPFT bodies the reference decodes; the per-stream tag sequence
equals the scope program's store log (vgpu.hpp:269-271, test_vgpu.cpp:273-281);
circular wrap keeps the tail (test_acceptance.cpp:104-147); unwrapped clocks
are monotone; the instrumented tcgen05 GEMM computes the same C as the plain
one and as cuBLAS."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def P1():
    from paper_2505_21661_b200 import p1
    return p1


@pytest.mark.parametrize("cap,iters", [(64, 3), (64, 20), (48, 20), (256, 30)])
def test_selftest_buffer_decodes_to_store_log(oracle, reference, cap, iters):
    import torch
    p1 = P1()
    ctas, warps = 5, 4
    stride = p1.stream_stride(cap)
    prof = torch.zeros(ctas * warps * stride, dtype=torch.uint8, device="cuda")
    timing = torch.zeros(ctas * 32, dtype=torch.uint8, device="cuda")
    p1.selftest(prof.data_ptr(), ctas, warps, cap, iters, timing.data_ptr())
    torch.cuda.synchronize()
    body = prof.cpu().numpy()
    img = p1.kpft_v1(body, ctas * warps)
    strategy = 0  # circular
    dec = oracle.decode_kpft(img, cap, strategy)
    log = p1.selftest_store_log(iters)
    tail = log[-cap:] if len(log) > cap else log
    for s, d in enumerate(dec):
        assert d["block_index"] == s // warps and d["warp_group"] == s % warps
        assert d["dropped_records"] == max(0, len(log) - cap)
        got = [((int(t) >> 31) & 1, (int(t) >> 12) & 0x7FFFF) for t in d["records"]["tag"]]
        assert got == tail
        u = oracle.unwrap_clock(d["records"]["payload"])
        assert np.all(np.diff(u.astype(np.int64)) >= 0)
    # the reference itself (oracle/_ref) reads the image and replays it, and
    # the C restatement agrees
    r = reference.replay_kpft(img, cap, strategy, P1().SELFTEST_LABELS, 33)
    assert len(r.events) > 0
    assert len(oracle.replay_kpft(img, cap, strategy, P1().SELFTEST_LABELS, 33).events) \
        == len(r.events)
    t = timing.cpu().numpy().view(P1().CTA_TIMING_DTYPE)
    assert np.all(t["gt_end"] >= t["gt_start"]) and np.all(t["streams"] == warps)


def test_selftest_buffer_through_gpu_decoder(ctx, oracle):
    """P1 body left in HBM -> P2 decoder in place (no host round trip)."""
    import torch
    from paper_2505_21661_b200 import trace as T
    p1 = P1()
    ctas, warps, cap, iters = 37, 8, 64, 40
    stride = p1.stream_stride(cap)
    prof = torch.zeros(ctas * warps * stride, dtype=torch.uint8, device="cuda")
    p1.selftest(prof.data_ptr(), ctas, warps, cap, iters)
    ctx.set_plan(T.BufferPlan(cap, T.BufferStrategy.Circular, p1.SELFTEST_LABELS))
    ev = torch.empty(ctas * warps * cap * 32, dtype=torch.uint8, device="cuda")
    ne, w = ctx.replay_device(prof.data_ptr(), prof.numel(), ctas * warps, 33,
                              ev.data_ptr(), ctas * warps * cap, 0x2)
    o = oracle.replay_body(prof.cpu().numpy(), ctas * warps, cap, 0,
                           p1.SELFTEST_LABELS, 33)
    assert ne == len(o.events)
    assert np.array_equal(ev[:ne * 32].cpu().numpy().view(O.EVENT_DTYPE), o.events)


def test_record_cost_is_small():
    import torch
    p1 = P1()
    n, warps = 4096, 4
    c0 = torch.zeros(warps, dtype=torch.int64, device="cuda")
    c1 = torch.zeros(warps, dtype=torch.int64, device="cuda")
    p1.record_cost(n, warps, False, c0.data_ptr())
    p1.record_cost(n, warps, True, c1.data_ptr())
    torch.cuda.synchronize()
    per_record = (c1.float().mean() - c0.float().mean()).item() / (2 * n)
    assert 0 < per_record < 40, per_record


# M % 256 == 0: the CTA-pair kernel (cta_group::2); M = 384: the single-CTA one
@pytest.mark.parametrize("shape", [(256, 512, 128), (1024, 1024, 2048), (384, 768, 192),
                                   (2048, 2048, 4096)])
def test_gemm_matches_cublas_and_instrumented_is_identical(oracle, shape):
    import torch
    p1 = P1()
    M, N, K = shape
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, generator=g, device="cuda").to(torch.bfloat16)
    C0 = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    C1 = torch.empty_like(C0)
    p1.gemm(A.data_ptr(), B.data_ptr(), C0.data_ptr(), M, N, K, False)
    ctas = p1.gemm_ctas(M, N)
    prof = torch.zeros(p1.gemm_profile_bytes(M, N), dtype=torch.uint8, device="cuda")
    p1.gemm(A.data_ptr(), B.data_ptr(), C1.data_ptr(), M, N, K, True, prof.data_ptr())
    torch.cuda.synchronize()
    ref = (A.float() @ B.float().T)
    err = (C0.float() - ref).abs().max().item()
    assert err <= 2e-2 * ref.abs().max().item(), err   # bf16 output rounding
    assert torch.equal(C0, C1)
    img = p1.kpft_v1(prof.cpu().numpy(), ctas * p1.GEMM_WARPS)
    r = oracle.replay_kpft(img, p1.GEMM_SLOTS, 0, p1.GEMM_LABELS, 0)
    # the GPU decoder on the device-resident profile (circular buffers: the
    # slots past each stream's surviving records hold older records)
    T = __import__("paper_2505_21661_b200.trace", fromlist=["trace"])
    ctx = T.Context(0)
    ctx.set_plan(T.BufferPlan(p1.GEMM_SLOTS, T.BufferStrategy.Circular, p1.GEMM_LABELS))
    n_streams = ctas * p1.GEMM_WARPS
    ev = torch.empty(n_streams * p1.GEMM_SLOTS * 32, dtype=torch.uint8, device="cuda")
    ne, w = ctx.replay_device(prof.data_ptr(), prof.numel(), n_streams, 0,
                              ev.data_ptr(), n_streams * p1.GEMM_SLOTS)
    assert ne == len(r.events)
    assert (w.dropped_heads, w.truncated_tails, w.flagged_preconditions,
            w.malformed_groups) == (r.dropped_heads, r.truncated_tails,
                                    r.flagged_preconditions, r.malformed_groups)
    gev = ev[: ne * 32].cpu().numpy().view(T.EVENT_DTYPE)
    assert np.array_equal(gev, r.events)
    # the stall scopes are sync scopes, not wait markers: nothing malformed
    assert w.malformed_groups == 0
    st = oracle.region_stats(r.events, p1.GEMM_LABELS)
    labels = {s.label for s in st}
    assert {"mma.issue", "tma.issue", "epi.ld", "epi.st", "tile"} <= labels


def test_pass_helpers_place_the_reference_records(oracle):
    """wgpf_dev::Scope / AsyncOp (the instrumentation pass as source helpers,
    instrument.hpp:145-153) store exactly the hand-instrumented program's
    records: same tags in the same order, and the body decodes."""
    import torch
    p1 = P1()
    ctas, warps, cap, iters = 3, 4, 64, 9
    stride = p1.stream_stride(cap)
    a = torch.zeros(ctas * warps * stride, dtype=torch.uint8, device="cuda")
    b = torch.zeros_like(a)
    c = torch.zeros_like(a)
    p1.selftest(a.data_ptr(), ctas, warps, cap, iters)
    p1.selftest_auto(b.data_ptr(), ctas, warps, cap, iters)
    p1.selftest_capi(c.data_ptr(), ctas, warps, cap, iters)  # C-style device API
    torch.cuda.synchronize()
    dc = oracle.decode_kpft(p1.kpft_v1(c.cpu().numpy(), ctas * warps), cap, 0)
    da = oracle.decode_kpft(p1.kpft_v1(a.cpu().numpy(), ctas * warps), cap, 0)
    db = oracle.decode_kpft(p1.kpft_v1(b.cpu().numpy(), ctas * warps), cap, 0)
    log = p1.selftest_store_log(iters)
    tail = log[-cap:] if len(log) > cap else log
    for x, y, z in zip(da, db, dc):
        assert np.array_equal(x["records"]["tag"], y["records"]["tag"])
        assert np.array_equal(x["records"]["tag"], z["records"]["tag"])
        assert (x["block_index"], x["warp_group"]) == (z["block_index"], z["warp_group"])
        got = [((int(t) >> 31) & 1, (int(t) >> 12) & 0x7FFFF) for t in y["records"]["tag"]]
        assert got == tail
