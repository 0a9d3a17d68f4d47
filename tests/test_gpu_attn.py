"""Config 3: the instrumented warp-specialised tcgen05 attention kernel
(csrc_p1/attn_tcgen05.cu).  Numerics against a torch fp32 softmax attention
(tolerance stated per test), the instrumented output bit-identical to the
plain one, its device profile decoded on the GPU bit-exactly against the CPU
oracle, and the overlap analysis (analyze_critical_path, perfmodel.hpp:317-501,
and the role overlap counters) on that trace equal to the oracle's."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

# bf16 inputs, fp32 softmax / accumulate, P rounded to bf16 before PV, bf16
# output: |O - O_ref| <= ATOL + RTOL |O_ref| against the fp32 reference
ATOL, RTOL = 2e-2, 2e-2


def P1():
    from paper_2505_21661_b200 import p1
    return p1


def ref_attention(q, k, v, scale=None):
    import torch
    scale = q.shape[-1] ** -0.5 if scale is None else scale
    s = (q.float() @ k.float().transpose(-1, -2)) * scale
    return torch.softmax(s, dim=-1) @ v.float()


def inputs(BH, S, seed=0, scale_q=1.0):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = (torch.randn(BH, S, 128, generator=g, device="cuda") * scale_q).to(torch.bfloat16)
    k = torch.randn(BH, S, 128, generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn(BH, S, 128, generator=g, device="cuda").to(torch.bfloat16)
    return q, k, v


def run(q, k, v, stages=2, instrument=False, prof=None, timing=None):
    import torch
    BH, S, _ = q.shape
    o = torch.empty_like(q)
    P1().attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), BH, S,
                   kv_stages=stages, instrument=instrument,
                   profile_ptr=prof.data_ptr() if prof is not None else 0,
                   timing_ptr=timing.data_ptr() if timing is not None else 0)
    torch.cuda.synchronize()
    return o


def close(o, ref):
    err = (o.float() - ref).abs()
    bad = err > ATOL + RTOL * ref.abs()
    return not bool(bad.any()), err.max().item()


@pytest.mark.parametrize("stages", [1, 2])
@pytest.mark.parametrize("BH,S,scale_q", [(1, 256, 1.0), (2, 512, 1.0), (3, 1024, 4.0),
                                          (1, 2048, 0.25)])
def test_attention_matches_fp32_reference(BH, S, scale_q, stages):
    q, k, v = inputs(BH, S, seed=BH * 7 + S, scale_q=scale_q)
    o = run(q, k, v, stages)
    ok, err = close(o, ref_attention(q, k, v))
    assert ok, err


def test_attention_structured_inputs():
    """Q = 0 -> uniform softmax -> O = column means of V (the PV path alone);
    one-hot V (V[key, d] = [key % 128 == d]) -> O[:, d] = sum of the softmax
    weights of keys = d (mod 128): pins the P column <-> key mapping."""
    import torch
    BH, S = 2, 512
    q, k, v = inputs(BH, S, seed=3)
    o = run(torch.zeros_like(q), k, v)
    ok, err = close(o, v.float().mean(dim=1, keepdim=True).expand_as(o))
    assert ok, err
    key = torch.arange(S, device="cuda")
    onehot = (key[:, None] % 128 == torch.arange(128, device="cuda")[None, :])
    v1 = onehot.to(torch.bfloat16).expand(BH, S, 128).contiguous()
    o = run(q, k, v1)
    ok, err = close(o, ref_attention(q, k, v1))
    assert ok, err


def test_attention_is_deterministic():
    """GEMM0 of tile j+1 is issued behind GEMM1 of tile j into the TMEM columns
    GEMM1 reads P from: any ordering race would show as run-to-run noise."""
    import torch
    q, k, v = inputs(16, 2048, seed=5, scale_q=2.0)
    for stages in (1, 2):
        o0 = run(q, k, v, stages)
        for _ in range(3):
            assert torch.equal(run(q, k, v, stages), o0)


def test_attention_rejects_bad_shapes():
    import torch
    q = torch.zeros(1, 384, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(RuntimeError):
        run(q, q, q)


@pytest.mark.parametrize("stages", [1, 2])
def test_instrumented_attention_trace(ctx, oracle, stages):
    """Instrumented == plain bit for bit; the device profile decodes on the
    GPU exactly as the oracle decodes it; GPU overlap analysis == oracle."""
    import torch
    from paper_2505_21661_b200 import trace as T
    p1 = P1()
    BH, S = 4, 2048
    q, k, v = inputs(BH, S, seed=11)
    o0 = run(q, k, v, stages)
    ctas = BH * S // 256
    prof = torch.zeros(p1.attn_profile_bytes(BH, S), dtype=torch.uint8, device="cuda")
    timing = torch.zeros(ctas * 32, dtype=torch.uint8, device="cuda")
    o1 = run(q, k, v, stages, True, prof, timing)
    assert torch.equal(o0, o1)
    n_streams = ctas * p1.ATTN_WARPS
    body = prof.cpu().numpy()
    hdr = body.reshape(n_streams, -1)[:, :16].copy().view(np.uint32)
    assert np.array_equal(hdr[:, 0], np.repeat(np.arange(ctas), p1.ATTN_WARPS))
    assert np.array_equal(hdr[:, 1], np.tile(np.arange(p1.ATTN_WARPS), ctas))
    nkv = S // 128
    assert np.all(hdr[:2 * 10:10, 2] == 4 * nkv)        # producers: 4 per tile
    assert np.all(hdr[2:10, 2] == 8 * nkv)              # consumers: 8 per tile

    want = oracle.replay_body(body, n_streams, p1.ATTN_SLOTS, 0, p1.ATTN_LABELS, 0)
    ctx.set_plan(T.BufferPlan(p1.ATTN_SLOTS, T.BufferStrategy.Circular, p1.ATTN_LABELS))
    ev = torch.empty(n_streams * p1.ATTN_SLOTS * 32, dtype=torch.uint8, device="cuda")
    ne, w = ctx.replay_device(prof.data_ptr(), prof.numel(), n_streams, 0,
                              ev.data_ptr(), n_streams * p1.ATTN_SLOTS)
    assert ne == len(want.events)
    assert (w.dropped_heads, w.truncated_tails, w.flagged_preconditions,
            w.malformed_groups) == (want.dropped_heads, want.truncated_tails,
                                    want.flagged_preconditions, want.malformed_groups)
    gev = ev[: ne * 32].cpu().numpy().view(T.EVENT_DTYPE)
    assert np.array_equal(gev, want.events)

    edges = p1.ATTN_BARRIER_EDGES
    got = ctx.critical_path(gev, edges, gate_by_block=True,
                            on_device_ptr=ev.data_ptr(), n_events=ne)
    exp = oracle.critical_path(want.events, p1.ATTN_LABELS, edges, gate_by_block=True)
    for key in ("stages", "mean", "steady", "wg", "binding", "cycle", "period"):
        assert got[key] == exp[key], key
    assert set(got["stages"]) >= {"GEMM0.c0", "Softmax.c1", "Load V"}
    roles = p1.ATTN_ROLE_OF_WARP
    assert ctx.overlap(gev, roles) == oracle.overlap(want.events, roles)
