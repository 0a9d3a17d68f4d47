"""Launch the config-2 GEMM alone (ncu target): plain, then instrumented."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_21661_b200 import p1
M = N = K = 8192
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
c = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
prof = torch.zeros(p1.gemm_profile_bytes(M, N), dtype=torch.uint8, device="cuda")
for instr in (False, False, True):
    p1.gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, instr, prof.data_ptr() if instr else 0)
torch.mm(a, b.T)
torch.cuda.synchronize()
