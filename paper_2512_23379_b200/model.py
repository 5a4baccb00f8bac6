"""Device-resident DiT denoiser (both modes) driven through the C-ABI kernels.

One `DeviceDenoiser` owns bf16 weights (transposed, K-major), fp32 vectors and
a workspace sized for one chunk geometry (L_c frames x T tokens/frame). A
denoise step is the reference's `Denoiser.forward` (net.py:244-276) laid out
as fused kernels:

  patchify(Eq.1) -> in-proj GEMM (+bias, +per-frame temb/pos row-add)
  per layer:  norm/AdaLN -> QKV GEMM (+3D RoPE epilogue) -> flash attention
              -> O GEMM (+gate * residual) -> LN -> cross-Q GEMM -> short-KV
              attention over per-chunk cond K/V -> cross-O GEMM (+residual)
              -> norm/AdaLN -> FFN1 GEMM (+bias, GELU) -> FFN2 GEMM (+bias, gate*residual)
  final norm/AdaLN -> out GEMM -> unpatchify + DDIM update (+ target x0 store)

ftlk mode reproduces the reference exactly (additive sinusoidal time/pos,
affine pre-LNs, heads of any width); wan mode adds 3D RoPE, AdaLN modulation
+ gates and 2x2 spatial patch tokens ("wan-shape extension").
"""

import math

import numpy as np
import torch

from . import ops
from .config import NetConfig, param_shapes
from .errors import ConfigError
from .rope import rope3d_tables

TIME_SCALE = 1000.0  # net.py:24


def round8(n):
    return (n + 7) // 8 * 8


def sinusoid(positions, dim):
    """[sin | cos] table, frequency denominator max(half-1, 1) (net.py:200-206); float64 host."""
    pos = np.asarray(positions, dtype=np.float64).reshape(-1)
    half = dim // 2
    freq = np.exp(-math.log(10000.0) * np.arange(half, dtype=np.float64) / max(half - 1, 1))
    ang = pos[:, None] * freq[None, :]
    return np.concatenate([np.sin(ang), np.cos(ang)], axis=1)


class DeviceWeights:
    """bf16 W^T matrices [N, round8(K)] + fp32 vectors on one device."""

    def __init__(self, cfg: NetConfig, device):
        self.cfg = cfg
        self.device = torch.device(device)
        self.mats = {}   # name -> (tensor [N, Kp], K)
        self.vecs = {}   # name -> fp32 tensor

    # -------- construction
    @classmethod
    def from_host(cls, cfg: NetConfig, params: dict, device):
        """params: name -> float64 ndarray in reference layout (in, out)."""
        self = cls(cfg, device)
        for name, shape in param_shapes(cfg):
            arr = np.asarray(params[name], dtype=np.float64)
            if arr.shape != tuple(shape):
                raise ConfigError("param %s has shape %s, expected %s" % (name, arr.shape, shape))
            if len(shape) == 2 and not name.endswith(".mod"):
                K, N = shape
                wt = torch.zeros(N, round8(K), dtype=torch.bfloat16)
                wt[:, :K] = torch.from_numpy(arr.T.copy()).to(torch.bfloat16)
                self.mats[name] = (wt.to(self.device), K)
            else:
                self.vecs[name] = torch.from_numpy(arr).to(torch.float32).to(self.device)
        self._fuse()
        return self

    @classmethod
    def synthetic(cls, cfg: NetConfig, device, seed=200):
        """Random-init weights of the named shape generated ON DEVICE (counter-based
        normal, same scaling rule as ParamStore.init: N(0,1)/sqrt(fan_in), gains 1,
        biases 0). Used for the 14B-shape benchmark, where a host fp64 init would
        need 105 GiB."""
        self = cls(cfg, device)
        for idx, (name, shape) in enumerate(param_shapes(cfg)):
            if len(shape) == 2 and not name.endswith(".mod"):
                K, N = shape
                wt = torch.zeros(N, round8(K), dtype=torch.bfloat16, device=self.device)
                if round8(K) == K:
                    ops.fill_normal_(wt, seed * 1000003 + idx, 1.0 / math.sqrt(K))
                else:
                    tmp = torch.empty(N, K, dtype=torch.bfloat16, device=self.device)
                    ops.fill_normal_(tmp, seed * 1000003 + idx, 1.0 / math.sqrt(K))
                    wt[:, :K] = tmp
                self.mats[name] = (wt, K)
            elif name.endswith(".mod"):
                t = torch.empty(shape, dtype=torch.float32, device=self.device)
                ops.fill_normal_(t, seed * 1000003 + idx, 1.0 / math.sqrt(shape[-1]))
                self.vecs[name] = t
            elif name.endswith(".g"):
                self.vecs[name] = torch.ones(shape, dtype=torch.float32, device=self.device)
            else:
                self.vecs[name] = torch.zeros(shape, dtype=torch.float32, device=self.device)
        self._fuse()
        return self

    def _fuse(self):
        """Concatenate q|k|v and cross k|v weights so each is one GEMM."""
        cfg = self.cfg
        for i in range(cfg.layers):
            p = "layers.%d." % i
            self.mats[p + "self.wqkv"] = (torch.cat([self.mats[p + "self.w" + c][0] for c in "qkv"], 0).contiguous(),
                                          cfg.model_dim)
            self.mats[p + "cross.wkv"] = (torch.cat([self.mats[p + "cross.w" + c][0] for c in "kv"], 0).contiguous(),
                                          cfg.model_dim)
            for c in "qkv":
                del self.mats[p + "self.w" + c]
            for c in "kv":
                del self.mats[p + "cross.w" + c]
        if cfg.mode == "wan":
            # per-layer modulation offsets stacked [layers, 6m]
            self.vecs["layers.mod"] = torch.stack(
                [self.vecs["layers.%d.mod" % i].reshape(-1) for i in range(cfg.layers)]).contiguous()

    def cross_wq_io(self, i):
        """Layer i's cross query projection in the reference (in, out) layout (the transpose of
        the stored W^T), cached: the B operand of the tensor-core fold At = kbd . Wq^T."""
        cache = self.__dict__.setdefault("_wq_io", {})
        if i not in cache:
            wt, K = self.mats["layers.%d.cross.wq" % i]
            cache[i] = wt[:, :K].t().contiguous()
        return cache[i]

    def nbytes(self):
        return sum(t.numel() * t.element_size() for t, _ in self.mats.values()) + \
            sum(t.numel() * t.element_size() for t in self.vecs.values())


class DeviceDenoiser:
    """Denoiser bound to device weights and one chunk geometry.

    Geometry: chunk_len L_c frames, motion_len L_m, latent grid (H, W)
    (ftlk: H = W = 1). Token count L = L_c * (H/ph) * (W/pw). With a
    communicator of world g > 1 the step runs Ulysses sequence parallel
    (dist.py): this rank owns tokens [start, start + Ls) of the padded chunk."""

    def __init__(self, weights: DeviceWeights, chunk_len, motion_len, latent_hw=(1, 1), stream=None, comm=None,
                 fold_cross=True, fold_band=True):
        from .dist import LocalComm, ShardPlan
        cfg = weights.cfg
        self.cfg, self.w = cfg, weights
        self.dev = weights.device
        self.Lc, self.Lm = int(chunk_len), int(motion_len)
        if not (0 <= self.Lm < self.Lc):
            raise ConfigError("motion_len must satisfy 0 <= L_m < L_c")
        self.H, self.W = (int(latent_hw[0]), int(latent_hw[1])) if cfg.mode == "wan" else (1, 1)
        self.ph, self.pw = (cfg.patch[1], cfg.patch[2]) if cfg.mode == "wan" else (1, 1)
        if self.H % self.ph or self.W % self.pw:
            raise ConfigError("latent grid must be divisible by the patch")
        self.gh, self.gw = self.H // self.ph, self.W // self.pw
        self.T = self.gh * self.gw
        self.L = self.Lc * self.T
        self.comm = comm if comm is not None else LocalComm()
        self.plan = ShardPlan(self.L, self.comm.world, self.comm.rank)
        self.hpr = self.plan.heads_per_rank(cfg.heads)
        m, ff = cfg.model_dim, cfg.ff_dim
        self.n_cond = self.Lc * (cfg.audio_tokens if cfg.mode == "wan" else 1) + 1
        d = self.dev
        bf, f32 = torch.bfloat16, torch.float32
        L, Lp, Ls, g = self.L, self.plan.L_pad, self.plan.Ls, self.plan.world
        hw = self.hpr * cfg.head_dim
        F = self.Lc + 1  # per-frame tables carry one extra (padding) frame
        self.kin = round8(cfg.in_features)
        self.ko = round8(cfg.out_features)
        self.buf = {
            "tok": torch.zeros(Lp, self.kin, dtype=bf, device=d),
            "h": torch.empty(Ls, m, dtype=f32, device=d),
            "u": torch.empty(Ls, m, dtype=bf, device=d),
            "qkv": torch.empty(Ls, 3 * m, dtype=bf, device=d),     # Ulysses send layout
            "ao": torch.empty(Ls, m, dtype=bf, device=d),
            "ff": torch.empty(Ls, ff, dtype=bf, device=d),
            "x0loc": torch.empty(Ls, self.ko, dtype=f32, device=d),
            "cond_in": torch.zeros(self.n_cond, round8(max(cfg.cond_dim, cfg.latent_dim)), dtype=bf, device=d),
            "cond": torch.empty(self.n_cond, m, dtype=f32, device=d),
            "cond_bf": torch.empty(self.n_cond, m, dtype=bf, device=d),
            "ckv": torch.empty(cfg.layers, self.n_cond, 2 * m, dtype=bf, device=d),
            "tfeat": torch.empty(F, m, dtype=bf, device=d),
            "temb": torch.empty(F, m, dtype=f32, device=d),
            "temb_act": torch.empty(F, m, dtype=bf, device=d),
            "e0": torch.empty(F, 6 * m, dtype=f32, device=d),
        }
        # folded cross-attention (wan): the projections fold through the chunk's fixed K/V
        # -> two m x (H*J) GEMMs per layer instead of two m x m ones. The fold runs on the
        # tensor cores over block-diagonal K / V operands (zero off the diagonal); At rows are in
        # the SEG_SOFTMAX tile order, so the logits GEMM's epilogue does the per-head softmax (no
        # fp32 logits round trip, no separate softmax pass)
        self.fold = cfg.mode == "wan" and self.n_cond <= 48 and fold_cross and m % 8 == 0
        if self.fold:
            self.J = round8(self.n_cond)
            HJ = cfg.heads * self.J
            self.fold_band = fold_band   # K loops of the fold GEMMs over the head bands only
            spt = 256 // self.J
            at_rows = (cfg.heads + spt - 1) // spt * 256
            self.buf["xat"] = torch.zeros(cfg.layers, at_rows, m, dtype=bf, device=d)
            self.buf["xbt"] = torch.empty(cfg.layers, m, HJ, dtype=bf, device=d)
            self.buf["xp"] = torch.empty(Ls, HJ, dtype=bf, device=d)
            self.buf["xkbd"] = torch.zeros(at_rows, m, dtype=bf, device=d)
            self.buf["xvbd"] = torch.zeros(HJ, m, dtype=bf, device=d)
        # caller-owned kernel scratch (the library keeps none): the flash kernel's KV-split
        # workspace and the split-K tail counters of the long-K residual GEMMs; every launch of
        # this denoiser is ordered on its stream, so one copy each serves all of them
        self.attn_ws = ops.attention_workspace(Lp, Lp, self.hpr, cfg.head_dim, d) if self.L > 128 else None
        self.buf["tail_ctr"] = torch.zeros(ops.A.TAIL_COUNTER_WORDS, dtype=torch.int32, device=d)
        self.peer = g > 1 and getattr(self.comm, "peer", False)
        if self.peer:
            # symmetric receive buffers: the producers' epilogues store into them over NVLink
            c = self.comm
            self.buf["qkv_recv"] = c.sym("qkv_recv", (Lp, 3 * hw), bf, d)     # [src][Ls][3][hpr][hd]
            self.buf["ao_recv"] = c.sym("ao_recv", (g * Ls, hw), bf, d)       # [src head group][Ls][hw]
            self.buf["x0tok"] = c.sym("x0tok", (Lp, self.ko), f32, d)
            r = self.plan.rank
            self._qkv_peers = [a + r * Ls * 3 * hw * 2 for a in c.addrs("qkv_recv")]
            self._ao_peers = [a + r * Ls * hw * 2 for a in c.addrs("ao_recv")]
            self._x0_peers = [a + r * Ls * self.ko * 4 for a in c.addrs("x0tok")]
        elif g > 1:
            self.buf["qkv_recv"] = torch.empty(Lp, 3 * hw, dtype=bf, device=d)
            self.buf["attn_full"] = torch.empty(Lp, hw, dtype=bf, device=d)
            self.buf["x0tok"] = torch.empty(Lp, self.ko, dtype=f32, device=d)
        else:
            self.buf["x0tok"] = self.buf["x0loc"]
        self.pos = torch.from_numpy(sinusoid(np.arange(F), m)).to(f32).to(d)  # chunk-relative frames
        self.rope = None
        if cfg.mode == "wan":
            self.rope_host = rope3d_tables(F, self.gh, self.gw, cfg.head_dim, cfg.rope_theta)
            self.rope = ops.RopeTables(self.rope_host, self.gh, self.gw, d)
        self._frame_cache = {}
        self.scale = 1.0 / math.sqrt(cfg.head_dim)
        self.stream = stream

    # ------------------------------------------------------------ per-frame vectors
    def frame_vectors(self, frame_t):
        """Per-frame time conditioning for a frame_t vector, cached (the ladder
        repeats every chunk). ftlk: rowvec[f] = temb[f] + pos[f] (net.py:229-232).
        wan: mods[l, f] = silu(temb)@tproj + b + layer.mod (6 x m), final[f] = final.mod + temb[f].
        One extra frame (t = 0) backs the Ulysses padding tokens."""
        key = tuple(float(t) for t in np.asarray(frame_t, dtype=np.float64).reshape(-1))
        hit = self._frame_cache.get(key)
        if hit is not None:
            return hit
        cfg, B, W = self.cfg, self.buf, self.w
        m = cfg.model_dim
        F = self.Lc + 1
        tf = torch.from_numpy(sinusoid(np.asarray(key + (0.0,)) * TIME_SCALE, m)).to(torch.bfloat16).to(self.dev)
        B["tfeat"].copy_(tf)
        wt, _ = W.mats["time.w"]
        out = {}
        if cfg.mode == "ftlk":
            rv = torch.empty(F, m, dtype=torch.float32, device=self.dev)
            ops.gemm(B["tfeat"], wt, rv, "rowadd_f32", bias=W.vecs["time.b"], group_vec=self.pos, rows_per_group=1,
                     stream=self.stream)
            out["rowvec"] = rv
        else:
            ops.gemm(B["tfeat"], wt, B["temb"], "f32", bias=W.vecs["time.b"], stream=self.stream)
            ops.silu_to_bf16(B["temb"], B["temb_act"], stream=self.stream)
            ops.gemm(B["temb_act"], W.mats["tproj.w"][0], B["e0"], "f32", bias=W.vecs["tproj.b"],
                     stream=self.stream)
            mods = torch.empty(cfg.layers, F, 6 * m, dtype=torch.float32, device=self.dev)
            ops.add_bcast(B["e0"], W.vecs["layers.mod"], mods, stream=self.stream)
            fin = torch.empty(F, 1, 2 * m, dtype=torch.float32, device=self.dev)
            # final.mod (2, m) + temb[f] broadcast over the 2 slots
            ops.add_bcast(W.vecs["final.mod"].reshape(1, 2 * m),
                          torch.cat([B["temb"], B["temb"]], 1).contiguous(), fin, stream=self.stream)
            out["mods"] = mods
            out["final"] = fin.view(F, 2 * m)
        self._frame_cache[key] = out
        return out

    # ------------------------------------------------------------ conditioning (once per chunk)
    def stage_cond(self, signal, reference, k=0):
        """Host half of the conditioning: driving window + reference token written
        (bf16) into pinned staging buffer k (two, so chunk c+1 stages while c copies)."""
        cfg = self.cfg
        nsig = self.n_cond - 1
        stages = getattr(self, "_cond_stage", None)
        if stages is None:
            stages = [torch.zeros(self.buf["cond_in"].shape, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
            self._cond_stage = stages
        st = stages[k]
        if cfg.mode == "ftlk":
            sig = torch.as_tensor(np.asarray(signal, dtype=np.float64).reshape(self.Lc, 1), dtype=torch.float32)
            ref = torch.as_tensor(np.asarray(reference, dtype=np.float64).reshape(1, -1), dtype=torch.float32)
        else:
            sig = torch.as_tensor(np.asarray(signal, dtype=np.float32).reshape(nsig, cfg.audio_dim))
            ref_lat = np.asarray(reference, dtype=np.float64).reshape(cfg.latent_dim, -1)
            ref = torch.as_tensor(ref_lat.mean(axis=1).reshape(1, -1), dtype=torch.float32)
        st.zero_()
        st[:nsig, :sig.shape[1]].copy_(sig.to(torch.bfloat16))
        st[nsig:, :ref.shape[1]].copy_(ref.to(torch.bfloat16))

    def copy_cond_in(self, k=0):
        """H2D of staging buffer k into the device cond input (stream-ordered)."""
        self.buf["cond_in"].copy_(self._cond_stage[k], non_blocking=True)

    def upload_cond(self):
        """Device half: cond input -> cond tokens (sig + frame pos ; ref) and the
        per-layer cross-attention K|V (net.py:233-237). Capturable in a CUDA graph."""
        with ops.nvtx("cond + cross K/V fold"):
            self._upload_cond()

    def _upload_cond(self):
        cfg, B, W = self.cfg, self.buf, self.w
        nsig = self.n_cond - 1
        ci = B["cond_in"]
        A = cfg.audio_tokens if cfg.mode == "wan" else 1
        ops.gemm(ci[:nsig], W.mats["sig.w"][0], B["cond"][:nsig], "rowadd_f32", bias=W.vecs["sig.b"],
                 group_vec=self.pos, rows_per_group=A, M=nsig, K=W.mats["sig.w"][1], lda=ci.stride(0),
                 stream=self.stream)
        ops.gemm(ci[nsig:], W.mats["ref.w"][0], B["cond"][nsig:], "f32", bias=W.vecs["ref.b"],
                 M=1, K=W.mats["ref.w"][1], lda=ci.stride(0), stream=self.stream)
        ops.cast_f32_bf16(B["cond"], B["cond_bf"], stream=self.stream)
        for i in range(cfg.layers):
            ops.gemm(B["cond_bf"], W.mats["layers.%d.cross.wkv" % i][0], B["ckv"][i], "bf16", stream=self.stream)
            if self.fold:
                # At = (scale * blockdiag K) . Wq^T and Bt = Wo^T . (blockdiag V)^T: two tensor-core
                # GEMMs over the zero-padded block-diagonal operands; each tile's K loop covers only
                # its rows' head bands (kbd rows in the SEG_SOFTMAX tile order: 256 // J heads per
                # 256-row tile; vbd rows head-major, J per head)
                ops.xattn_blockdiag(B["ckv"][i], B["xkbd"], B["xvbd"], self.n_cond, cfg.heads, cfg.head_dim, self.J,
                                    self.scale, k_tiled=True, stream=self.stream)
                fl = 2.0 * cfg.heads * self.J * cfg.head_dim * cfg.model_dim   # non-zero blocks only
                band_k = (0, self.J, 256, 256 // self.J, cfg.head_dim) if self.fold_band else None
                band_v = (1, self.J, 0, 0, cfg.head_dim) if self.fold_band else None
                ops.gemm(B["xkbd"], W.cross_wq_io(i), B["xat"][i], "bf16", band=band_k, stream=self.stream,
                         algo_flops=fl)
                ops.gemm(W.mats["layers.%d.cross.wo" % i][0], B["xvbd"], B["xbt"][i], "bf16", band=band_v,
                         stream=self.stream, algo_flops=fl)

    def prepare_cond(self, signal, reference):
        """cond = [sig tokens + frame pos ; ref token] and per-layer cross K|V
        (once per chunk: cond does not change across the sampler's steps)."""
        self.stage_cond(signal, reference, 0)
        self.copy_cond_in(0)
        self.upload_cond()

    # ------------------------------------------------------------ one denoise step
    def step(self, motion, z, reference, fv, x0_out=None, ddim=None, stacked=None):
        """One Denoiser.forward on device. motion [L_m, D, H, W], z [L_c-L_m, D, H, W],
        reference [D, H, W] (fp32 device). Writes x0 tokens to buf['x0tok'] (all L
        tokens on every rank); if x0_out is given, also unpatchifies the target frames
        (and applies the DDIM update to z when ddim=(a_i, s_i, a_n, s_n)).
        stacked: an explicit composite [L_c][2D+1][H][W] (f32 device) instead of the canonical
        one assembled from motion / z / reference (any z_mask / z_cond rows)."""
        cfg, B, W = self.cfg, self.buf, self.w
        m, H_, hd = cfg.model_dim, cfg.heads, cfg.head_dim
        L, T, s = self.L, self.T, self.stream
        pl = self.plan
        s0, Ls, g, hpr = pl.start, pl.Ls, pl.world, self.hpr
        hw = hpr * hd
        D = cfg.latent_dim
        if stacked is not None:
            ops.patchify_stacked(stacked, self.ph, self.pw, B["tok"][:L], stream=s)
        else:
            ops.patchify(motion, z, reference, self.Lm, self.Lc, D, self.H, self.W, self.ph, self.pw, B["tok"][:L],
                         stream=s)
        h = B["h"]
        tok = B["tok"][s0:s0 + Ls]
        wan = cfg.mode == "wan"
        if wan:
            ops.gemm(tok, W.mats["in.w"][0], h, "f32", bias=W.vecs["in.b"], K=W.mats["in.w"][1], M=Ls,
                     lda=self.kin, stream=s)
        else:
            ops.gemm(tok, W.mats["in.w"][0], h, "rowadd_f32", bias=W.vecs["in.b"], group_vec=fv["rowvec"],
                     rows_per_group=T, row_offset=s0, K=W.mats["in.w"][1], M=Ls, lda=self.kin, stream=s)
        u, qkv, ao, ffb = B["u"], B["qkv"], B["ao"], B["ff"]
        for i in range(cfg.layers):
            ops.nvtx_push("layer %d" % i)
            p = "layers.%d." % i
            if wan:
                md = fv["mods"][i]  # [L_c + 1, 6m]
                ops.norm_modulate(h, u, shift=md[:, 0:m], scale=md[:, m:2 * m], rows_per_group=T, row_offset=s0,
                                  stream=s)
            else:
                ops.norm_modulate(h, u, gamma=W.vecs[p + "ln1.g"], beta=W.vecs[p + "ln1.b"], stream=s)
            ops.gemm(u, W.mats[p + "self.wqkv"][0], qkv, "qkv_rope", heads=H_, head_dim=hd, heads_per_rank=hpr,
                     row_offset=s0, rope=self.rope, peers=self._qkv_peers if self.peer else None, stream=s)
            if self.peer:
                # all-to-all #1 rode the QKV epilogue; #2 rides the FMHA epilogue
                rq = B["qkv_recv"]
                self.comm.barrier(s)
                ops.attention_scatter(rq[:, 0:hw], rq[:, hw:2 * hw], rq[:, 2 * hw:], hpr, hd, pl.L_pad, L,
                                      self.scale, self._ao_peers, Ls, hw, workspace=self.attn_ws, stream=s)
                self.comm.barrier(s)
                o_in = dict(a=B["ao_recv"], M=Ls, K=m, lda=hw, a_chunks=g, a_chunk_stride=Ls * hw)
            elif g == 1:
                ops.attention(qkv[:, 0:m], qkv[:, m:2 * m], qkv[:, 2 * m:], ao, H_, hd, L, L, self.scale,
                              workspace=self.attn_ws, stream=s)
                o_in = dict(a=ao)
            else:
                rq, af = B["qkv_recv"], B["attn_full"]
                self.comm.all_to_all(rq, qkv, stream=s)                       # heads <- sequence
                ops.attention(rq[:, 0:hw], rq[:, hw:2 * hw], rq[:, 2 * hw:], af, hpr, hd, pl.L_pad, L, self.scale,
                              workspace=self.attn_ws, stream=s)
                self.comm.all_to_all(ao, af, stream=s)                        # sequence <- heads
                o_in = dict(a=ao, M=Ls, K=m, lda=hw, a_chunks=g, a_chunk_stride=Ls * hw)
            if wan:
                ops.gemm(o_in.pop("a"), W.mats[p + "self.wo"][0], h, "resid_f32", group_vec=md[:, 2 * m:3 * m],
                         rows_per_group=T, row_offset=s0, stream=s, **o_in)
            else:
                ops.gemm(o_in.pop("a"), W.mats[p + "self.wo"][0], h, "resid_f32", stream=s, **o_in)
            ops.norm_modulate(h, u, gamma=W.vecs[p + "ln2.g"], beta=W.vecs[p + "ln2.b"], stream=s)
            if self.fold:   # P = softmax_seg(U.At^T) (logits GEMM, softmax in its epilogue); h += P.Bt^T
                ops.xattn_logits_softmax(u, B["xat"][i], B["xp"], H_, self.J, self.n_cond, stream=s)
                ops.gemm(B["xp"], B["xbt"][i], h, "resid_f32", stream=s)
            else:
                ops.gemm(u, W.mats[p + "cross.wq"][0], qkv[:, 0:m], "bf16", stream=s)
                ckv = B["ckv"][i]
                ops.attention(qkv[:, 0:m], ckv[:, 0:m], ckv[:, m:], ao, H_, hd, Ls, self.n_cond, self.scale, stream=s)
                ops.gemm(ao, W.mats[p + "cross.wo"][0], h, "resid_f32", stream=s)
            if wan:
                ops.norm_modulate(h, u, shift=md[:, 3 * m:4 * m], scale=md[:, 4 * m:5 * m], rows_per_group=T,
                                  row_offset=s0, stream=s)
            else:
                ops.norm_modulate(h, u, gamma=W.vecs[p + "ln3.g"], beta=W.vecs[p + "ln3.b"], stream=s)
            ops.gemm(u, W.mats[p + "ffn.w1"][0], ffb, "gelu_bf16", bias=W.vecs[p + "ffn.b1"], stream=s)
            tail = B["tail_ctr"]
            if wan:
                ops.gemm(ffb, W.mats[p + "ffn.w2"][0], h, "resid_f32", bias=W.vecs[p + "ffn.b2"],
                         group_vec=md[:, 5 * m:6 * m], rows_per_group=T, row_offset=s0, stream=s, tail_counters=tail)
            else:
                ops.gemm(ffb, W.mats[p + "ffn.w2"][0], h, "resid_f32", bias=W.vecs[p + "ffn.b2"], stream=s,
                         tail_counters=tail)
            ops.nvtx_pop()
        if wan:
            fm = fv["final"]
            ops.norm_modulate(h, u, shift=fm[:, 0:m], scale=fm[:, m:2 * m], rows_per_group=T, row_offset=s0, stream=s)
        else:
            ops.norm_modulate(h, u, gamma=W.vecs["final.g"], beta=W.vecs["final.b"], stream=s)
        ops.gemm(u, W.mats["out.w"][0], B["x0loc"], "f32", bias=W.vecs["out.b"],
                 peers=self._x0_peers if self.peer else None, stream=s)
        x0t = B["x0tok"]
        if self.peer:
            self.comm.barrier(s)                       # all-gather rode the out-projection epilogue
        elif g > 1:
            self.comm.all_gather(x0t, B["x0loc"], stream=s)
        if x0_out is not None:
            ops.unpatch_ddim(x0t[:L, :cfg.out_features], self.Lm, self.Lc, D, self.H, self.W, self.ph, self.pw, z,
                             x0_out, coeffs=ddim, stream=s)
        return x0t[:L]

    # ------------------------------------------------------------ full-chunk output (reference forward)
    def tokens_to_frames(self, x0t):
        """x0 tokens [L, out_features] -> (L_c, D, H, W) float tensor (device)."""
        cfg = self.cfg
        x = x0t[:self.L, :cfg.out_features].reshape(self.Lc, self.gh, self.gw, cfg.latent_dim, self.ph, self.pw)
        return x.permute(0, 3, 1, 4, 2, 5).reshape(self.Lc, cfg.latent_dim, self.H, self.W)

    # ------------------------------------------------------------ the few-step sampler on device
    def sample(self, motion, reference, z, plan, x0_out, trace=None):
        """DDIM ladder (diffusion.py:202-237) entirely on device. motion/reference/z
        are device fp32; z is updated in place; x0_out [L_c-L_m, D, H, W] receives
        the final x0 (the chunk's target latents)."""
        ts = plan.timesteps
        coeffs = plan.ddim_coefficients()
        for i, t in enumerate(ts):
            frame_t = np.where(np.arange(self.Lc) < self.Lm, 0.0, float(t))
            fv = self.frame_vectors(frame_t)
            if trace is not None:
                trace.append((float(t), z.clone()))
            with ops.nvtx("ladder step %d (t=%.3g)" % (i, t)):
                self.step(motion, z, reference, fv, x0_out=x0_out, ddim=coeffs[i] if i + 1 < len(ts) else None)
            if trace is not None:
                trace[-1] = trace[-1] + (x0_out.clone(),)
        return x0_out
