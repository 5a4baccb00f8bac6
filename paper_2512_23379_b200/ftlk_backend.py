"""`b200` operator backend: the reference's kernel table (`backends/__init__.py:44-51`)
served by the sm_100a kernels.

Same function names and NumPy-in / NumPy-out contract as
`ftlk.backends.reference` (float64 2-D C-contiguous arrays in, fresh arrays
out), so `FTLK_BACKEND=b200` can plug it into the reference's table. Each
call moves its operands to the device (bf16) and back, so this table exists
for operator-level parity, not speed — the performance path is the
device-resident `Denoiser` (net.py mirror). Tolerance is bf16, not the
1e-12 of the reference's Cython parity test. Backward kernels are training
only and out of scope: they raise NotImplementedError.
"""

import math

import numpy as np
import torch

from . import ops
from .errors import ConfigError

NAME = "b200"
_DEV = "cuda"


def _bf(x):
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 2:
        raise ConfigError("operator inputs must be 2-d arrays")
    return torch.as_tensor(x, dtype=torch.float32).to(_DEV).to(torch.bfloat16)


def _wt(w):
    w = np.asarray(w, dtype=np.float64)
    K, N = w.shape
    Kp = (K + 7) // 8 * 8
    wt = torch.zeros(N, Kp, dtype=torch.bfloat16)
    wt[:, :K] = torch.as_tensor(w.T.copy(), dtype=torch.float32).to(torch.bfloat16)
    return wt.to(_DEV), K


def _rows(x):
    """bf16 activations padded to a multiple of 8 columns (TMA row stride)."""
    x = np.asarray(x, dtype=np.float64)
    M, K = x.shape
    Kp = (K + 7) // 8 * 8
    t = torch.zeros(M, Kp, dtype=torch.bfloat16, device=_DEV)
    t[:, :K] = torch.as_tensor(x, dtype=torch.float32).to(_DEV).to(torch.bfloat16)
    return t, K


def dense_forward(x, w, b):
    """x @ w + b (backends/reference.py:17-18)."""
    xt, K = _rows(x)
    wt, _ = _wt(w)
    out = torch.empty(xt.shape[0], wt.shape[0], dtype=torch.float32, device=_DEV)
    ops.gemm(xt, wt, out, "f32", bias=torch.as_tensor(np.asarray(b), dtype=torch.float32).to(_DEV),
             M=xt.shape[0], K=K, lda=xt.stride(0))
    return out.double().cpu().numpy()


def gelu_forward(x):
    """tanh GELU (backends/reference.py:28-31)."""
    xt = _bf(x).contiguous()
    y = torch.empty_like(xt)
    ops.gelu_bf16(xt, y)
    return y.double().cpu().numpy()


def layernorm_forward(x, gamma, beta):
    """(y, mean, rstd) (backends/reference.py:41-46)."""
    x = np.asarray(x, dtype=np.float64)
    xd = torch.as_tensor(x, dtype=torch.float32).to(_DEV)
    M, N = x.shape
    y = torch.empty(M, N, dtype=torch.bfloat16, device=_DEV)
    mean = torch.empty(M, dtype=torch.float32, device=_DEV)
    rstd = torch.empty(M, dtype=torch.float32, device=_DEV)
    ops.norm_modulate(xd, y, gamma=torch.as_tensor(gamma, dtype=torch.float32).to(_DEV),
                      beta=torch.as_tensor(beta, dtype=torch.float32).to(_DEV), mean_out=mean, rstd_out=rstd)
    return y.double().cpu().numpy(), mean.double().cpu().numpy(), rstd.double().cpu().numpy()


def mha_forward(xq, xkv, wq, wk, wv, wo, heads):
    """(y, cache) (backends/reference.py:77-92), cache = (q, k, v, p, ctx) as the reference's:
    the flash kernel never materialises the probabilities, so p comes from a separate
    device pass (ops.attention_probs) over the same bf16 q and k."""
    m = np.asarray(xq).shape[1]
    hd = m // heads

    def proj(x, w):
        xt, K = _rows(x)
        wt, _ = _wt(w)
        o = torch.empty(xt.shape[0], wt.shape[0], dtype=torch.bfloat16, device=_DEV)
        ops.gemm(xt, wt, o, "bf16", M=xt.shape[0], K=K, lda=xt.stride(0))
        return o

    q, k, v = proj(xq, wq), proj(xkv, wk), proj(xkv, wv)
    ctx = torch.empty_like(q)
    ops.attention(q, k, v, ctx, heads, hd, q.shape[0], k.shape[0], 1.0 / math.sqrt(hd))
    y = dense_forward(ctx.double().cpu().numpy(), wo, np.zeros(np.asarray(wo).shape[1]))
    probs = ops.attention_probs(q, k, heads, hd, q.shape[0], k.shape[0], 1.0 / math.sqrt(hd))
    split = [t.double().cpu().numpy().reshape(t.shape[0], heads, hd).transpose(1, 0, 2) for t in (q, k, v)]
    return y, (split[0], split[1], split[2], probs.double().cpu().numpy(), ctx.double().cpu().numpy())


def _training_only(*_a, **_k):
    raise NotImplementedError("backward kernels are training-only and out of scope for the b200 backend")


dense_backward = gelu_backward = layernorm_backward = mha_backward = _training_only
