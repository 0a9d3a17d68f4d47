"""Step-by-step GPU diagnostics (each step in its own process under a timeout).

    python scripts/diag.py <step>
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def log(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, flush=True)


def main(step):
    import numpy as np
    log("import torch")
    import torch
    log("torch", torch.__version__, torch.cuda.is_available())
    from oracle import oracle as O
    from oracle import synth as S
    from paper_2505_21661_b200 import _build, trace as T
    log("build")
    _build.build()
    log("lib", _build.LIB)
    ctx = T.Context(0)
    log("ctx ok")
    orc = O.Oracle()
    from conftest import load_fixture
    data, slots, strategy, labels, cost, _ = load_fixture("fa3_vanilla")
    plan = T.BufferPlan(slots, T.BufferStrategy(strategy), labels)
    want = orc.replay_kpft(data, slots, strategy, labels, cost)
    if step == "general":
        r = ctx.replay_image_bytes(data, plan, cost, flags=0x4)
        log("general events", len(r.events), np.array_equal(r.events, want.events))
    elif step == "fast_nostats":
        r = ctx.replay_image_bytes(data, plan, cost, flags=0x8)
        log("fast events", len(r.events), np.array_equal(r.events, want.events))
    elif step == "fast":
        r = ctx.replay_image_bytes(data, plan, cost, flags=0)
        log("fast events", len(r.events), np.array_equal(r.events, want.events))
        st = ctx.stats()
        log("stats", {k: (v.count, v.mean) for k, v in st.items()})
    elif step == "exact":
        r = ctx.replay_image_bytes(data, plan, cost, flags=0x2)
        log("exact events", len(r.events), np.array_equal(r.events, want.events))
        st = ctx.stats()
        log("stats", {k: (v.count, v.mean) for k, v in st.items()})
    elif step == "synth":
        n = 4096
        ctx.set_plan(T.BufferPlan(S.CAP, T.BufferStrategy.Flush, S.MIXED_LABELS))
        body = torch.empty(n * S.stream_stride(), dtype=torch.uint8, device="cuda")
        ctx.synth_body(body.data_ptr(), 0, S.MIXED_FULL_LONG - n // 2, n,
                       S.MIXED_FULL_LONG)
        torch.cuda.synchronize()
        cpu = S.mixed_body(S.MIXED_FULL_LONG - n // 2, n, S.MIXED_FULL_LONG)
        log("synth equal", np.array_equal(body.cpu().numpy(), cpu))
        ev = torch.empty(n * 128 * 32, dtype=torch.uint8, device="cuda")
        for flags in (0x4, 0x8, 0):
            ne, w = ctx.replay_device(body.data_ptr(), body.numel(), n, 33,
                                      ev.data_ptr(), n * 128, flags)
            o = orc.replay_body(cpu, n, S.CAP, 1, S.MIXED_LABELS, 33)
            got = ev[:ne * 32].cpu().numpy().view(O.EVENT_DTYPE)
            log("flags", flags, "ne", ne, len(o.events), np.array_equal(got, o.events),
                ctx.last_profile())
    log("done")


if __name__ == "__main__":
    main(sys.argv[1])
