"""One small launch of every kernel family of libftb2.so, meant for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per gpurun call):

    compute-sanitizer --tool memcheck python scripts/sanitize_kernels.py

compute-sanitizer is CLOSED on this GPU pool (profiles/r02_sanitizer.md); the out-of-bounds
checks run as guard-band tests instead (tests/test_guard_bands_gpu.py), and this sweep runs
plain as a smoke of every kernel family.

GEMM (single CTA, CTA pair, residual + split-K tail, QKV + RoPE, segment softmax, block-diagonal
band), flash attention (+ KV-split + combine), short-KV and CUDA-core attention, attention
probabilities, norm / AdaLN,
patchify / unpatch + DDIM, causal conv (per-tap, dx-reuse pair / vertical, fused norm, halo, RGB
head), VAE norm / upsample, codec, barrier self-test. Shapes are the smallest that reach each
kernel's code paths (ragged tiles included)."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_23379_b200 import _capi as A  # noqa: E402
from paper_2512_23379_b200 import ops  # noqa: E402
from paper_2512_23379_b200.rope import rope3d_tables  # noqa: E402


def bf(*shape, scale=1.0):
    return (torch.randn(*shape, device="cuda") * scale).to(torch.bfloat16)


def main():
    torch.manual_seed(0)
    dev = torch.device("cuda")
    # ---------------- GEMM
    for (M, N, K) in [(300, 512, 256), (100, 192, 128), (1, 64, 16)]:
        a, w = bf(M, K), bf(N, K, scale=0.05)
        ops.gemm(a, w, torch.empty(M, N, device=dev), "f32", bias=torch.randn(N, device=dev))
        ops.gemm(a, w, torch.empty(M, N, device=dev, dtype=torch.bfloat16), "gelu_bf16")
        h = torch.randn(M, N, device=dev)
        ops.gemm(a, w, h, "resid_f32", group_vec=torch.randn(3, N, device=dev), rows_per_group=(M + 2) // 3)
        ops.gemm(a, w, h, "resid_f32", variant=6)
    M, N, K = 47 * 256 - 100, 512, 8192    # split-K tail: 94 tiles -> 20 tail tiles in 3 K-slices
    a, w = bf(M, K), bf(N, K, scale=0.01)
    ctr = torch.zeros(A.TAIL_COUNTER_WORDS, dtype=torch.int32, device=dev)
    ops.gemm(a, w, torch.randn(M, N, device=dev), "resid_f32", tail_counters=ctr)
    heads, hd, gh, gw, F = 4, 64, 4, 6, 3
    L = F * gh * gw
    rope = ops.RopeTables(rope3d_tables(F + 1, gh, gw, hd, 10000.0), gh, gw, dev)
    u = bf(L, heads * hd)
    ops.gemm(u, bf(3 * heads * hd, heads * hd, scale=0.05), torch.empty(L, 3 * heads * hd, device=dev,
             dtype=torch.bfloat16), "qkv_rope", heads=heads, head_dim=hd, heads_per_rank=heads // 2, rope=rope)
    J, segs = 40, 13
    spt = 256 // J
    at = bf((segs + spt - 1) // spt * 256, 256, scale=0.05)
    ops.xattn_logits_softmax(bf(300, 256), at, torch.empty(300, segs * J, device=dev, dtype=torch.bfloat16),
                             segs, J, 37)
    kv = bf(37, 2 * heads * hd)
    kbd = torch.zeros(256, heads * hd, device=dev, dtype=torch.bfloat16)
    vbd = torch.zeros(heads * J, heads * hd, device=dev, dtype=torch.bfloat16)
    ops.xattn_blockdiag(kv, kbd, vbd, 37, heads, hd, J, 0.1, k_tiled=True)
    ops.gemm(kbd, bf(heads * hd, heads * hd).t().contiguous(), torch.empty(256, heads * hd, device=dev,
             dtype=torch.bfloat16), "bf16", band=(0, J, 256, spt, hd))
    # ---------------- attention
    for (Lq, Lk, H, d) in [(700, 700, 4, 128), (300, 260, 2, 64)]:
        q, k, v = bf(Lq, H * d), bf(Lk, H * d), bf(Lk, H * d)
        ops.attention(q, k, v, torch.empty_like(q), H, d, Lq, Lk, 1 / math.sqrt(d), impl=0)
    Lq, H, d = 2600, 148 * 3 // 2, 64      # items > SMs: the KV-split tail + combine
    q = bf(Lq, H * d)
    ws = ops.attention_workspace(Lq, Lq, H, d, dev)
    ops.attention(q, q, q, torch.empty_like(q), H, d, Lq, Lq, 0.125, impl=0, workspace=ws)
    q, kv = bf(500, 4 * 128), bf(37, 8 * 128)
    ops.attention(q, kv[:, :512], kv[:, 512:], torch.empty_like(q), 4, 128, 500, 37, 0.088)
    ops.attention(bf(9, 32), bf(10, 32), bf(10, 32), torch.empty(9, 32, device=dev, dtype=torch.bfloat16), 2, 16,
                  9, 10, 0.25)
    ops.attention_probs(bf(9, 32), bf(10, 32), 2, 16, 9, 10, 0.25)
    # ---------------- norm / elementwise
    x = torch.randn(300, 1536, device=dev)
    ops.norm_modulate(x, torch.empty(300, 1536, device=dev, dtype=torch.bfloat16),
                      scale=torch.randn(3, 1536, device=dev), shift=torch.randn(3, 1536, device=dev),
                      rows_per_group=100)
    ops.norm_modulate(torch.randn(50, 5120, device=dev), torch.empty(50, 5120, device=dev, dtype=torch.bfloat16),
                      gamma=torch.ones(5120, device=dev), beta=torch.zeros(5120, device=dev))
    z = torch.randn(2, 16, 8, 12, device=dev)
    mo = torch.randn(1, 16, 8, 12, device=dev)
    ref = torch.randn(16, 8, 12, device=dev)
    tok = torch.empty(3 * 24, 136, device=dev, dtype=torch.bfloat16)
    ops.patchify(mo, z, ref, 1, 3, 16, 8, 12, 2, 2, tok)
    x0 = torch.randn(72, 64, device=dev)
    ops.unpatch_ddim(x0, 1, 3, 16, 8, 12, 2, 2, z, torch.empty_like(z), coeffs=(0.5, 0.5, 0.75, 0.25))
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    ops.count_nonfinite(x0, flag)
    # ---------------- VAE convs + norms
    from paper_2512_23379_b200.vae import DeviceVAEDecoder, VAEConfig
    for base in (32, 96):
        dec = DeviceVAEDecoder(VAEConfig(z_dim=16, base_dim=base), dev, params=None, seed=1, rgb8=True)
        dec.decode_device_tensor(torch.randn(2, 16, 3, 17, device=dev), torch.cuda.current_stream())
    # ---------------- barrier protocol (concurrent ranks in one cooperative launch)
    fl = torch.zeros(16, dtype=torch.int32, device=dev)
    ep = torch.zeros(4, dtype=torch.int32, device=dev)
    dat = torch.zeros(400, dtype=torch.int32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    A.call("ftb_peer_barrier_selftest", 4, 100, A.ptr(fl), A.ptr(ep), A.ptr(dat), A.ptr(err), 10.0, A.stream_ptr())
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    print("sanitize_kernels: all launches completed")


if __name__ == "__main__":
    main()
