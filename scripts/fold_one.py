"""One folded cross-attention weight prep at the 14B shape (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_23379_b200 import ops  # noqa: E402

m, H, hd, nc, J = 5120, 40, 128, 37, 40
dev = torch.device("cuda")
kv = torch.randn(nc, 2 * m, device=dev).to(torch.bfloat16)
wq = (torch.randn(m, m, device=dev) / 70).to(torch.bfloat16)
wo = (torch.randn(m, m, device=dev) / 70).to(torch.bfloat16)
at = torch.empty(H * J, m, device=dev, dtype=torch.bfloat16)
bt = torch.empty(m, H * J, device=dev, dtype=torch.bfloat16)
for _ in range(3):
    ops.xattn_fold(kv, wq, wo, at, bt, nc, H, hd, J, 0.088)
torch.cuda.synchronize()
print("ok")
