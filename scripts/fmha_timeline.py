"""Per-block softmax timeline of one flash-attention CTA (debug build with -DFTB_FMHA_TIMELINE,
loaded through FTB_LIB). Stamps per block j and tile t: 0 start, 1 S ready, 2 S loaded,
3 max done, 4 first-half exps, 5 PV(j-1) done, 6 P stored."""
import ctypes as C
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_23379_b200 import _capi as A  # noqa: E402
from paper_2512_23379_b200 import ops  # noqa: E402

L, H, hd = 10530, 40, 128
q, k, v = (torch.randn(L, H * hd, device="cuda").to(torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
impl = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for _ in range(2):
    ops.attention(q, k, v, o, H, hd, L, L, 1 / math.sqrt(hd), impl=impl)
torch.cuda.synchronize()
buf = np.zeros((2, 128, 8), dtype=np.int64)
fn = A.lib.ftb_debug_fmha_timeline
fn.argtypes = [C.c_void_p]
assert fn(buf.ctypes.data) == 0
n = (L + 127) // 128
for t in range(2):
    b = buf[t, 8:n - 4].astype(np.float64)
    period = np.diff(buf[t, 8:n - 4, 0]).mean()
    seg = lambda a, c: float(np.mean(b[:, c] - b[:, a]))  # noqa: E731
    print("tile %d: period %.0f clk | wait S %.0f | S load %.0f | max %.0f | exp half1 %.0f | wait PV(j-1) %.0f | "
          "store+exp half2 %.0f | tail %.0f" % (t, period, seg(0, 1), seg(1, 2), seg(2, 3), seg(3, 4), seg(4, 5),
                                                seg(5, 6), period - seg(0, 6)))
print("tile offset (t1 - t0 start) %.0f clk" % float(np.mean(buf[1, 8:n - 4, 0] - buf[0, 8:n - 4, 0])))
