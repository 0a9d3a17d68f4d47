import sys, os, statistics, torch, json
sys.path.insert(0, os.getcwd())
from paper_2505_21661_b200 import p1
M=N=K=8192
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
B = torch.randn(N, K, generator=g, device="cuda").to(torch.bfloat16)
C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
prof = torch.zeros(p1.gemm_profile_bytes(M, N), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(instr, n=20, fl=True):
    ts=[]
    for i in range(n):
        if fl: flush.zero_()
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); p1.gemm(A.data_ptr(),B.data_ptr(),C.data_ptr(),M,N,K,instr,prof.data_ptr() if instr else 0); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return ts
for _ in range(3): t(False,5); t(True,5)
res={}
for fl in (True, False):
  for r in range(3):
    a=t(False, fl=fl); b=t(True, fl=fl)
    res[f"fl{fl}_r{r}"]=(round(statistics.median(a),4), round(statistics.median(b),4), round(100*(statistics.median(b)/statistics.median(a)-1),2))
print(json.dumps(res))
