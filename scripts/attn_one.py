"""One FMHA launch at the 14B shape (L=10530, 40 heads, hd 128) for ncu: python scripts/attn_one.py IMPL"""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_23379_b200 import ops  # noqa: E402

impl = int(sys.argv[1]) if len(sys.argv) > 1 else 0
L, H, hd = 10530, 40, 128
q, k, v = (torch.randn(L, H * hd, device="cuda").to(torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
for _ in range(2):
    ops.attention(q, k, v, o, H, hd, L, L, 1 / math.sqrt(hd), impl=impl)
torch.cuda.synchronize()
print("ok", float(o.float().abs().mean()))
