"""Launch the attention kernel alone (ncu target): config-3 shape."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_21661_b200 import p1
BH, S = int(os.environ.get("BH", 256)), 8192
st = int(os.environ.get("STAGES", 1))
q, k, v = (torch.randn(BH, S, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
for i in range(2):
    p1.attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), BH, S, kv_stages=st)
torch.cuda.synchronize()
