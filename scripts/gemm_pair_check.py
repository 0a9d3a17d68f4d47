"""CTA-pair GEMM check: outputs vs torch.matmul on several shapes, the
instrumented twin identical, and plain / instrumented / single-CTA / cuBLAS
timings at 8192^3 (CUDA events, L2 flushed)."""
import os
import statistics
import subprocess
import sys
import json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def check():
    import torch
    from paper_2505_21661_b200 import p1
    for (M, N, K) in [(256, 256, 64), (256, 512, 128), (512, 768, 320), (1024, 1024, 2048),
                      (2048, 4096, 1024), (8192, 8192, 8192)]:
        g = torch.Generator(device="cuda").manual_seed(1)
        A = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
        B = torch.randn(N, K, generator=g, device="cuda").to(torch.bfloat16)
        C0 = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda")
        C1 = torch.full_like(C0, float("nan"))
        p1.gemm(A.data_ptr(), B.data_ptr(), C0.data_ptr(), M, N, K, False)
        prof = torch.zeros(p1.gemm_profile_bytes(M, N), dtype=torch.uint8, device="cuda")
        p1.gemm(A.data_ptr(), B.data_ptr(), C1.data_ptr(), M, N, K, True, prof.data_ptr())
        torch.cuda.synchronize()
        ref = A.float() @ B.float().T
        err = (C0.float() - ref).abs().max().item()
        print(json.dumps({"shape": [M, N, K], "ctas": p1.gemm_ctas(M, N), "err": err,
                          "refmax": ref.abs().max().item(),
                          "identical": bool(torch.equal(C0, C1))}), flush=True)


def timing():
    import torch
    from paper_2505_21661_b200 import p1
    M = N = K = 8192
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    prof = torch.zeros(p1.gemm_profile_bytes(M, N), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def t(fn, n=20):
        ts = []
        for i in range(n + 3):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)
    f = 2.0 * M * N * K
    plain = lambda: p1.gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, False)
    instr = lambda: p1.gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, True,
                            prof.data_ptr())

    def one(fn):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1)
    for _ in range(3):
        one(plain); one(instr)
    tp, ti, rat = [], [], []
    for _ in range(40):  # alternating launches: the ratio of neighbours
        a = one(plain); b = one(instr)
        tp.append(a); ti.append(b); rat.append(b / a)
    r = {"plain": {"ms": statistics.median(tp)}, "instr": {"ms": statistics.median(ti)},
         "cublas": {"ms": t(lambda: torch.matmul(A, B.T))}}
    for v in r.values():
        v["tflops"] = f / v["ms"] / 1e9
    r["ovh_pct"] = 100 * (statistics.median(rat) - 1)
    print(json.dumps({"single" if os.environ.get("WGPF_GEMM_SINGLE") == "1" else "pair": r}), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "check":
        check()
    else:
        timing()
