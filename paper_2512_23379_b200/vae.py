"""Causal 3D VAE decoder (wan mode), streaming with per-conv causal caches.

Build-defined "Wan-2.1-shaped" decoder (PAPER.md:151 names the Wan2.1 VAE;
the reference stands it in with an orthogonal codec, world.py:181-210):

  conv_in  CausalConv3d(z -> d0, 3x3x3)
  mid      ResBlock(d0) -> AttentionBlock(d0) -> ResBlock(d0)
           AttentionBlock(x) = x + proj(attn(qkv(rms(x))))  per frame, one head over the
           frame's h*w pixels (head_dim d0, scale 1/sqrt(d0)); qkv / proj are 1x1 convs
  stage i  (num_res_blocks+1) x ResBlock(in_i -> d_{i+1});
           i < 3: [time_conv CausalConv3d(C -> 2C, 3x1x1) -> frames x2]  (temporal_upsample[i])
                   nearest 2x spatial upsample -> Conv2d 3x3 (C -> C/2)
  head     RMSNorm -> SiLU -> CausalConv3d(d_last -> 3, 3x3x3) -> RGB
  ResBlock(x) = conv2(silu(rms2(conv1(silu(rms1(x)))))) + (x | conv1x1(x))

dims = base * [m_last] + base * reversed(mult) = [384, 384, 384, 192, 96] at base 96.
Every causal conv keeps the last 2 input frames of the previous chunk as its
cache (zeros at stream start), so decoding the chunks' target latents in
order equals one causal decode of the whole latent stream; each latent frame
yields 4 video frames (7 latents -> 28 frames per chunk).

Device layout: channel-last bf16 activations, convs are tcgen05 implicit GEMMs
(`ftb_conv3d_bf16`), norms/upsample are HBM-bound kernels. Weight layout on
the host is PyTorch's Conv3d (Cout, Cin, kt, kh, kw) float64.
"""

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi as A
from . import ops
from .errors import ConfigError
from .seeding import INIT, rng_for


@dataclass(frozen=True)
class VAEConfig:
    z_dim: int = 16
    base_dim: int = 96
    dim_mult: tuple = (1, 2, 4, 4)
    num_res_blocks: int = 2
    temporal_upsample: tuple = (True, True, False)
    mid_attention: bool = True

    @property
    def dims(self):
        m = tuple(self.dim_mult)
        return [self.base_dim * m[-1]] + [self.base_dim * u for u in reversed(m)]

    @property
    def time_factor(self):
        return 2 ** sum(bool(t) for t in self.temporal_upsample)

    @property
    def space_factor(self):
        return 2 ** (len(self.dim_mult) - 1)


def _conv(name, cin, cout, k):
    return [(name + ".w", (cout, cin) + tuple(k)), (name + ".b", (cout,))]


def _res(name, cin, cout):
    s = [(name + ".norm1.g", (cin,))] + _conv(name + ".conv1", cin, cout, (3, 3, 3))
    s += [(name + ".norm2.g", (cout,))] + _conv(name + ".conv2", cout, cout, (3, 3, 3))
    if cin != cout:
        s += _conv(name + ".shortcut", cin, cout, (1, 1, 1))
    return s


def vae_program(cfg: VAEConfig):
    """Ordered op list: (op, name, cin, cout) with op in
    conv_in | res | attn | time | resample | head; plus param shapes."""
    d = cfg.dims
    prog = [("conv_in", "conv_in", cfg.z_dim, d[0])]
    shapes = _conv("conv_in", cfg.z_dim, d[0], (3, 3, 3))
    for j in range(2):
        prog.append(("res", "mid.%d" % j, d[0], d[0]))
        shapes += _res("mid.%d" % j, d[0], d[0])
        if j == 0 and cfg.mid_attention:
            prog.append(("attn", "mid.attn", d[0], d[0]))
            shapes += [("mid.attn.norm.g", (d[0],))] + _conv("mid.attn.qkv", d[0], 3 * d[0], (1, 1, 1))
            shapes += _conv("mid.attn.proj", d[0], d[0], (1, 1, 1))
    n_up = len(cfg.dim_mult)
    for i in range(n_up):
        cin = d[i] // 2 if i > 0 else d[i]
        cout = d[i + 1]
        for j in range(cfg.num_res_blocks + 1):
            nm = "up.%d.res.%d" % (i, j)
            prog.append(("res", nm, cin, cout))
            shapes += _res(nm, cin, cout)
            cin = cout
        if i != n_up - 1:
            if cfg.temporal_upsample[i]:
                prog.append(("time", "up.%d.time" % i, cout, 2 * cout))
                shapes += _conv("up.%d.time" % i, cout, 2 * cout, (3, 1, 1))
            prog.append(("resample", "up.%d.resample" % i, cout, cout // 2))
            shapes += _conv("up.%d.resample" % i, cout, cout // 2, (1, 3, 3))
    prog.append(("head", "head", d[-1], 3))
    shapes += [("head.norm.g", (d[-1],))] + _conv("head.conv", d[-1], 3, (3, 3, 3))
    return prog, shapes


def init_vae_params(cfg: VAEConfig, seed: int) -> dict:
    """Host float64 params: conv weights N(0,1)/sqrt(fan_in), biases 0, gains 1."""
    rng = rng_for(seed, INIT, 1)
    _, shapes = vae_program(cfg)
    out = {}
    for name, shape in shapes:
        if name.endswith(".g"):
            out[name] = np.ones(shape)
        elif name.endswith(".b"):
            out[name] = np.zeros(shape)
        else:
            fan_in = int(np.prod(shape[1:]))
            out[name] = rng.standard_normal(shape) / np.sqrt(fan_in)
    return out


class _ConvW:
    """Device conv weights W^T [Cout_pad][taps*Cin] bf16 + bias, and its causal cache."""

    def __init__(self, w, b, device, pad_cout_to=None):
        cout, cin, kt, kh, kw = w.shape
        self.cin, self.cout, self.k = cin, cout, (kt, kh, kw)
        rows = pad_cout_to or cout
        wt = np.zeros((rows, kt * kh * kw * cin))
        wt[:cout] = np.transpose(w, (0, 2, 3, 4, 1)).reshape(cout, -1)
        self.wt = torch.as_tensor(wt).to(torch.bfloat16).to(device).contiguous()
        bb = np.zeros(rows)
        bb[:cout] = b
        self.b = torch.as_tensor(bb, dtype=torch.float32).to(device)
        self.cache = None

    @classmethod
    def synthetic(cls, shape, device, seed, pad_cout_to=None):
        self = cls.__new__(cls)
        cout, cin, kt, kh, kw = shape
        self.cin, self.cout, self.k = cin, cout, (kt, kh, kw)
        rows = pad_cout_to or cout
        self.wt = torch.zeros(rows, kt * kh * kw * cin, dtype=torch.bfloat16, device=device)
        tmp = torch.empty(cout, kt * kh * kw * cin, dtype=torch.bfloat16, device=device)
        ops.fill_normal_(tmp, seed, 1.0 / np.sqrt(cin * kt * kh * kw))
        self.wt[:cout] = tmp
        self.b = torch.zeros(rows, dtype=torch.float32, device=device)
        self.cache = None
        return self


class DeviceVAEDecoder:
    """Streaming causal decoder on one device. `decode_device(z)` decodes one
    chunk of target latents [T, z_dim, h, w] and advances the causal caches.

    With a communicator of world g > 1 the decode is split spatially along the
    latent rows: conv_in runs on the full (replicated) latent, then
    rank r owns a contiguous slab of rows at every level (slabs double with each
    2x upsample). Before every 3x3 convolution the ranks swap their edge rows
    (one row per side at that level's resolution, all frames) with their
    neighbours; the conv kernel reads rows -1 / H_local from those halo buffers
    (zeros at the global edges), so the split decode equals the unsplit one.
    The causal caches of the halo rows travel with the caches of the slabs."""

    def __init__(self, cfg: VAEConfig, device, params=None, seed=0, rgb8=True, comm=None, fuse_norm=True,
                 head_gemm=True):
        from .dist import LocalComm
        self.cfg = cfg
        self.dev = torch.device(device)
        self.prog, shapes = vae_program(cfg)
        self.rgb8 = rgb8
        # RGB8 head as one 1x1 GEMM (27 taps x 3 channels as output rows) + a 27-tap gather
        # (ftb_conv3d_head_rgb8) instead of the N = 3 implicit-GEMM conv
        self.head_gemm = head_gemm
        # RMS norm + SiLU of a conv output folded into that conv's epilogue whenever one N tile
        # holds every channel of a pixel (Cout <= 192): the normalised bf16 tensor is written
        # straight into the next conv's input buffer (no fp32 re-read, no separate pass)
        # True / "all": conv1 -> norm2 and conv2 / resample -> next norm1 / head norm;
        # "conv1": only conv1 -> norm2 (no fp32 main output); False / "none": separate passes
        self.fuse_norm = {True: "all", False: "none"}.get(fuse_norm, fuse_norm)
        if self.fuse_norm not in ("all", "conv1", "none"):
            raise ConfigError("fuse_norm must be True/False/'all'/'conv1'/'none'")
        self.frames_per_latent = cfg.time_factor
        self.comm = comm if comm is not None else LocalComm()
        self.W, self.G = {}, {}
        for idx, (name, shape) in enumerate(shapes):
            if name.endswith(".g"):
                g = np.ones(shape) if params is None else params[name]
                self.G[name[:-2]] = torch.as_tensor(g, dtype=torch.float32).to(self.dev)
            elif name.endswith(".w"):
                base = name[:-2]
                pad = 32 if base == "head.conv" else None
                if params is None:
                    self.W[base] = _ConvW.synthetic(shape, self.dev, seed * 7919 + idx, pad)
                else:
                    self.W[base] = _ConvW(params[name], params[base + ".b"], self.dev, pad)
        self._geo = None
        self._host = {}

    @property
    def split(self):
        return self.comm.world > 1

    # ------------------------------------------------------------ buffers
    def _setup(self, T, h, w):
        key = (T, h, w)
        if self._geo == key:
            return
        self._geo = key
        from .dist import slab_rows
        g, r = self.comm.world, self.comm.rank
        sizes = slab_rows(h, g)
        self.sizes = sizes
        self.row0, self.rows = sum(sizes[:r]), sizes[r]
        geo = [dict(T=T, H=self.rows, W=w, C=0)]
        ups = 1
        for op, name, cin, cout in self.prog:
            cur = geo[-1]
            if op in ("conv_in", "res"):
                cur["C"] = max(cur["C"], cin, cout)
            elif op == "head":
                cur["C"] = max(cur["C"], cin)
            elif op == "time":
                cur["C"] = max(cur["C"], cin)
                geo.append(dict(T=2 * cur["T"], H=cur["H"], W=cur["W"], C=cin))
            elif op == "resample":
                cur["C"] = max(cur["C"], cin)
                ups = max(ups, cur["T"] * 4 * cur["H"] * cur["W"] * cin)
                geo.append(dict(T=cur["T"], H=2 * cur["H"], W=2 * cur["W"], C=cout, HC=cin))
        bf, f32 = torch.bfloat16, torch.float32
        levels = {}
        for l, gg in enumerate(geo):
            px, C = gg["T"] * gg["H"] * gg["W"], gg["C"]
            Tp = gg["T"] + 2
            levels[l] = dict(gg, x=torch.empty(px * C, dtype=f32, device=self.dev),      # residual stream
                             sc=torch.empty(px * C, dtype=f32, device=self.dev),     # 1x1 shortcut
                             h=torch.empty(px * C, dtype=bf, device=self.dev),       # conv1 output
                             xb=torch.empty(px * C, dtype=bf, device=self.dev),      # bf16 view of x
                             work=torch.empty(Tp * gg["H"] * gg["W"] * C, dtype=bf, device=self.dev),
                             work2=torch.empty(Tp * gg["H"] * gg["W"] * C, dtype=bf, device=self.dev))
            if self.split:  # halo rows (+2 cache frames) and contiguous edge-row send buffers
                row = gg["W"] * max(C, gg.get("HC", 0))
                if getattr(self.comm, "peer", False):
                    # symmetric receive buffers: the neighbours store their edge rows here over NVLink
                    top = self.comm.sym("vae_top%d" % l, (Tp * row,), bf, self.dev)
                    bot = self.comm.sym("vae_bot%d" % l, (Tp * row,), bf, self.dev)
                else:
                    top = torch.zeros(Tp * row, dtype=bf, device=self.dev)
                    bot = torch.zeros(Tp * row, dtype=bf, device=self.dev)
                levels[l].update(top=top, bot=bot, lvl=l,
                                 s_first=torch.empty(Tp * row, dtype=bf, device=self.dev),
                                 s_last=torch.empty(Tp * row, dtype=bf, device=self.dev))
        self.levels = levels
        self.attn = None
        if any(op == "attn" for op, *_ in self.prog):
            g0 = geo[0]
            C0, HWl, HW = g0["C"], g0["H"] * g0["W"], h * w
            HWp = (HW + 7) // 8 * 8   # GEMM operand rows 16-byte aligned
            npx0 = g0["T"] * HWl
            kv_shape = (g0["T"], h, w, 2 * C0)
            self.attn = dict(q=torch.empty(npx0, C0, dtype=bf, device=self.dev),
                             kv=torch.empty(npx0, 2 * C0, dtype=bf, device=self.dev),
                             vt=torch.empty(C0, HWp, dtype=bf, device=self.dev),
                             s=torch.empty(HWl, HWp, dtype=f32, device=self.dev),
                             p=torch.empty(HWl, HWp, dtype=bf, device=self.dev),
                             o=torch.empty(npx0, C0, dtype=bf, device=self.dev),
                             kv_full=None)
            if self.split:   # every rank needs every row's keys and values
                self.attn["kv_full"] = (self.comm.sym("vae_kv", kv_shape, bf, self.dev)
                                        if getattr(self.comm, "peer", False)
                                        else torch.empty(kv_shape, dtype=bf, device=self.dev))
        self.upbuf = torch.empty(ups, dtype=bf, device=self.dev)
        self.full0 = torch.empty(T * h * w * geo[0]["C"], dtype=f32, device=self.dev) if self.split else None
        last = levels[len(geo) - 1]
        npx = last["T"] * last["H"] * last["W"]
        self.out_rgb = torch.empty(npx * 3, dtype=torch.uint8, device=self.dev)
        self.out_f = torch.empty(npx * 32, dtype=f32, device=self.dev)
        self.frames_full = None
        if self.split:   # rank 0 receives every slab of the decoded frames (engine output)
            sf = last["H"] // self.rows
            full = (last["T"], h * sf, last["W"], 3 if self.rgb8 else 32)
            dt = torch.uint8 if self.rgb8 else f32
            self.px_sizes = [n * sf for n in sizes]
            self.frames_full = (self.comm.sym("vae_frames", full, dt, self.dev) if getattr(self.comm, "peer", False)
                                else torch.empty(full, dtype=dt, device=self.dev))
        for cw in self.W.values():
            cw.cache = None
            cw.hcache = None
        self.reset()

    def reset(self):
        """Zero the causal caches (stream start)."""
        for cw in self.W.values():
            if cw.cache is not None:
                cw.cache.zero_()
            if getattr(cw, "hcache", None) is not None:
                cw.hcache.zero_()

    # ------------------------------------------------------------ primitive wrappers
    OUT_F32, RESID_F32 = 16, 32

    def _exchange_halos(self, L, src, T_in, Cin, off=0):
        """Edge rows of `src` frames [0, T_in) -> neighbours; the neighbours' edge rows
        land in L['top'] / L['bot'] frames [off, off + T_in) (zeros at the global edges)."""
        H, W = L["H"], L["W"]
        row = W * Cin
        v = src[:T_in * H * row].view(T_in, H, row)
        first, last = L["s_first"][:T_in * row].view(T_in, row), L["s_last"][:T_in * row].view(T_in, row)
        first.copy_(v[:, 0])
        last.copy_(v[:, H - 1])
        top = L["top"][off * row:(off + T_in) * row].view(T_in, row)
        bot = L["bot"][off * row:(off + T_in) * row].view(T_in, row)
        if getattr(self.comm, "peer", False):   # stores into the neighbours' receive buffers + barrier
            self.comm.halo_store("vae_top%d" % L["lvl"], "vae_bot%d" % L["lvl"], off * row * 2, first, last, top,
                                 bot)
        else:
            self.comm.neighbor_exchange(first, last, top, bot)
        return L["top"][:(off + T_in) * row], L["bot"][:(off + T_in) * row]

    def _causal(self, cw, L, Cin, producer, out, out_ld, mode, resid=None, resid_ld=0, stream=None, halo=True,
                work_key="work", norm=None):
        """KT=3 causal conv on level L: cache -> work[0:2], producer fills
        work[2:] (None: a previous conv's fused-norm epilogue already did), (split: halo
        exchange of the new frames), conv, last 2 input frames -> cache (next chunk)."""
        T, H, W = L["T"], L["H"], L["W"]
        fr = H * W * Cin
        work = L[work_key][:(T + 2) * fr]
        if cw.cache is None:
            cw.cache = torch.zeros(2 * fr, dtype=torch.bfloat16, device=self.dev)
        work[:2 * fr].copy_(cw.cache)
        if producer is not None:
            producer(work[2 * fr:])
        halos = None
        if self.split and halo and cw.k[1] == 3:
            row = W * Cin
            if cw.hcache is None:
                cw.hcache = torch.zeros(2, 2 * row, dtype=torch.bfloat16, device=self.dev)
            # exchange the T new frames; the 2 cached halo frames come from this conv's halo cache
            tv, bv = self._exchange_halos(L, work[2 * fr:], T, Cin, off=2)
            tv[:2 * row].copy_(cw.hcache[0])
            bv[:2 * row].copy_(cw.hcache[1])
            cw.hcache[0].copy_(tv[T * row:(T + 2) * row])
            cw.hcache[1].copy_(bv[T * row:(T + 2) * row])
            halos = (tv, bv)
        self._conv(work, T + 2, H, W, Cin, cw, out, out_ld, 0, mode, resid, resid_ld, T, stream, halos,
                   allow_halo=halo, norm=norm)
        cw.cache.copy_(work[T * fr:(T + 2) * fr])

    def _conv(self, inp, T_in, H, W, Cin, cw, out, out_ld, t0, mode, resid, resid_ld, T_out, stream, halos=None,
              allow_halo=True, norm=None):
        kt, kh, kw = cw.k
        cout = cw.cout if (mode & 15) != 0 or cw.cout % 32 == 0 else cw.wt.shape[0]
        if self.split and allow_halo and kh == 3 and halos is None:   # non-causal 3x3 (resample)
            L = next(lv for lv in self.levels.values() if lv["H"] == H and lv["W"] == W and lv["T"] == T_in)
            halos = self._exchange_halos(L, inp, T_in, Cin)
        tag = "conv" if ops.PROFILE_DETAIL is None else "conv:%dx%dx%d %d->%d k%d%d%d" % (
            T_out, H, W, Cin, cw.cout, kt, kh, kw)
        if (mode & 15) == 2 and self.head_gemm and (kt, kh, kw) == (3, 3, 3) and Cin % 8 == 0:
            self._head_rgb8(inp, T_in, H, W, Cin, cw, out, t0, T_out, stream, halos)
            return
        if (kt, kh, kw) == (1, 1, 1) and mode == self.OUT_F32 and resid is None and cw.cout % 32 == 0:
            # 1x1x1 conv (resblock shortcut) = a plain GEMM over the pixels (the implicit-GEMM conv
            # ran it at ~60 TFLOP/s)
            npx = T_out * H * W
            a = inp[t0 * H * W * Cin:(t0 + T_out) * H * W * Cin].view(npx, Cin)
            tag = "conv" if ops.PROFILE_DETAIL is None else "conv:%dx%dx%d %d->%d k111 gemm" % (
                T_out, H, W, Cin, cw.cout)
            ops.gemm(a, cw.wt, out[:npx * out_ld].view(npx, out_ld)[:, :cw.cout], "f32", bias=cw.b[:cw.cout],
                     stream=stream, prof_kind=tag)
            return
        mode = mode | (A.CONV_VARIANT << 8)   # kernel selection of this call (0 = auto; A/B runs)
        with ops._Prof(tag, 2.0 * T_out * H * W * cw.cout * kt * kh * kw * Cin, 0.0, stream):
            if norm is not None:
                gamma, nout, write_main = norm
                nrm = A.ConvNorm(A.ptr(gamma), A.ptr(nout), cout, 1, int(write_main))
                A.call("ftb_conv3d_norm_bf16", A.ptr(inp), A.ptr(halos[0]) if halos else None,
                       A.ptr(halos[1]) if halos else None, T_in, H, W, Cin, A.ptr(cw.wt), cout, kt, kh, kw, t0,
                       A.ptr(cw.b), A.ptr(resid), resid_ld, A.ptr(out), out_ld, T_out, mode, C.byref(nrm),
                       A.stream_ptr(stream))
            elif halos is not None:
                A.call("ftb_conv3d_halo_bf16", A.ptr(inp), A.ptr(halos[0]), A.ptr(halos[1]), T_in, H, W, Cin,
                       A.ptr(cw.wt), cout, kt, kh, kw, t0, A.ptr(cw.b), A.ptr(resid), resid_ld, A.ptr(out), out_ld,
                       T_out, mode, A.stream_ptr(stream))
            else:
                A.call("ftb_conv3d_bf16", A.ptr(inp), T_in, H, W, Cin, A.ptr(cw.wt), cout, kt, kh, kw, t0,
                       A.ptr(cw.b), A.ptr(resid), resid_ld, A.ptr(out), out_ld, T_out, mode, A.stream_ptr(stream))

    def _head_rgb8(self, inp, T_in, H, W, Cin, cw, out, t0, T_out, stream, halos):
        if getattr(cw, "w_taps", None) is None:   # [81][Cin]: row tap*3 + c, tap = (dt*3+dy)*3+dx
            cw.w_taps = cw.wt[:3].reshape(3, 27, Cin).permute(1, 0, 2).reshape(81, Cin).contiguous()
        need = 81 * (T_in * H * W + (2 * T_in * W if halos else 0))
        ws = getattr(self, "_head_ws", None)
        if ws is None or ws.numel() < need:
            ws = torch.empty(need, dtype=torch.bfloat16, device=self.dev)
            self._head_ws = ws
        tag = "conv" if ops.PROFILE_DETAIL is None else "conv:%dx%dx%d %d->3 head gemm+gather" % (T_out, H, W, Cin)
        with ops._Prof(tag, 2.0 * T_out * H * W * 3 * 27 * Cin, 0.0, stream):
            A.call("ftb_conv3d_head_rgb8", A.ptr(inp), A.ptr(halos[0]) if halos else None,
                   A.ptr(halos[1]) if halos else None, T_in, H, W, Cin, A.ptr(cw.w_taps), A.ptr(cw.b), A.ptr(ws),
                   ws.numel(), A.ptr(out), T_out, t0, A.stream_ptr(stream))
        A.LAUNCHES[0] += T_in + (2 if halos is not None else 0)   # per-frame GEMMs (+ halos) + gather

    def _rms(self, x, npix, C, g, y, stream):
        fn = "ftb_rmsnorm_silu_f32" if x.dtype == torch.float32 else "ftb_rmsnorm_silu_bf16"
        with ops._Prof("vae_norm", 0.0, float(npix) * C * (x.element_size() + 2), stream):
            A.call(fn, A.ptr(x), npix, C, A.ptr(g), 1e-12, 1, A.ptr(y), A.stream_ptr(stream))

    # ------------------------------------------------------------ decode
    def decode_device_tensor(self, z, stream=None, gather=False):
        """z: device f32 [T, z_dim, h, w] -> device output (uint8 [T*tf, H, W, 3] if
        rgb8 else f32 [T*tf, H, W, 32] with channels 0..2 valid). With a split
        communicator the output is this rank's row slab [T*tf, H_local, W, .]; with
        gather=True every slab is collected into rank 0's full frames (returned on rank 0,
        None on the other ranks)."""
        with ops.nvtx("vae decode"):
            out = self._decode(z, stream)
        self.last_slab = out
        if not (gather and self.split):
            return out
        self.comm.gather_rows("vae_frames", self.frames_full, out, self.px_sizes, stream)
        return self.frames_full if self.comm.rank == 0 else None

    def _decode(self, z, stream=None):
        if z.dim() != 4 or z.shape[1] != self.cfg.z_dim:
            raise ConfigError("VAE input must be [T, z_dim, h, w]")
        T, _, h, w = z.shape
        self._setup(T, h, w)
        s = stream
        lv = self.levels
        F32, R32 = self.OUT_F32, self.RESID_F32
        l = 0
        cw = self.W["conv_in"]
        zc = self.cfg.z_dim
        if not self.split:
            self._causal(cw, lv[0], zc,
                         lambda dst: A.call("ftb_nchw_to_nhwc_bf16", A.ptr(z), T, zc, h, w, A.ptr(dst), zc,
                                            A.stream_ptr(s)),
                         lv[0]["x"], cw.cout, F32, stream=s)
        else:   # conv_in on the full (replicated) latent, then keep this rank's rows
            full = dict(T=T, H=h, W=w, work=self._full_work(T, h, w, zc))
            self._causal(cw, full, zc,
                         lambda dst: A.call("ftb_nchw_to_nhwc_bf16", A.ptr(z), T, zc, h, w, A.ptr(dst), zc,
                                            A.stream_ptr(s)),
                         self.full0, cw.cout, F32, stream=s, halo=False)
            C0 = cw.cout
            lv[0]["x"][:T * self.rows * w * C0].view(T, self.rows, w, C0).copy_(
                self.full0.view(T, h, w, C0)[:, self.row0:self.row0 + self.rows])
        pre = None   # (level, work key) whose frames [2:] already hold the next conv's normalised input
        prog = self.prog
        for i in range(1, len(prog)):
            op, name, cin, cout = prog[i]
            L = lv[l]
            T_, H_, W_ = L["T"], L["H"], L["W"]
            npx = T_ * H_ * W_
            x = L["x"]
            if op == "res":
                c1, c2 = self.W[name + ".conv1"], self.W[name + ".conv2"]
                if cin != cout:  # 1x1 shortcut of the block input
                    ops.cast_f32_bf16(x[:npx * cin], L["xb"][:npx * cin], stream=s)
                    self._conv(L["xb"], T_, H_, W_, cin, self.W[name + ".shortcut"], L["sc"], cout, 0, F32, None, 0,
                               T_, s)
                    resid = L["sc"]
                else:
                    resid = x
                prod1 = None if pre == (l, "work") else (
                    lambda dst: self._rms(x[:npx * cin], npx, cin, self.G[name + ".norm1"], dst, s))
                fr2 = H_ * W_ * cout
                if self.fuse_norm != "none" and cout <= 192:   # conv1 -> norm2 + SiLU -> conv2's input
                    self._causal(c1, L, cin, prod1, None, cout, 0, stream=s,
                                 norm=(self.G[name + ".norm2"], L["work2"][2 * fr2:], False))
                    prod2 = None
                else:
                    self._causal(c1, L, cin, prod1, L["h"], cout, 0, stream=s)
                    prod2 = (lambda dst: self._rms(L["h"][:npx * cout], npx, cout, self.G[name + ".norm2"], dst, s))
                # conv2 updates the fp32 residual stream in place (one thread reads and writes each pixel) and,
                # fused, writes the next block's (or the head's) normalised input
                nxt = self._next_norm(i, cout)
                self._causal(c2, L, cout, prod2, x, cout, F32 | R32, resid=resid, resid_ld=cout, stream=s,
                             work_key="work2",
                             norm=(nxt, L["work"][2 * fr2:], True) if nxt is not None else None)
                pre = (l, "work") if nxt is not None else None
            elif op == "attn":
                self._mid_attention(name, L, cin, s)
                pre = None
            elif op == "time":
                nxt = lv[l + 1]
                self._causal(self.W[name], L, cin, lambda dst: ops.cast_f32_bf16(x[:npx * cin], dst, stream=s),
                             nxt["x"], cin, 1 | F32, stream=s)
                l += 1
                pre = None
            elif op == "resample":
                up = self.upbuf[:npx * 4 * cin]
                with ops._Prof("vae_upsample", 0.0, float(npx) * cin * (4 + 4 * 2), s):
                    A.call("ftb_upsample2x_f32_bf16", A.ptr(x), T_, H_, W_, cin, A.ptr(up), A.stream_ptr(s))
                nxt = lv[l + 1]
                g = self._next_norm(i, cout)
                fr_n = nxt["H"] * nxt["W"] * cout
                self._conv(up, T_, 2 * H_, 2 * W_, cin, self.W[name], nxt["x"], cout, 0, F32, None, 0, T_, s,
                           norm=(g, nxt["work"][2 * fr_n:], True) if g is not None else None)
                l += 1
                pre = (l, "work") if g is not None else None
            elif op == "head":
                hw_ = self.W["head.conv"]
                prod = None if pre == (l, "work") else (
                    lambda dst: self._rms(x[:npx * cin], npx, cin, self.G["head.norm"], dst, s))
                if self.rgb8:
                    self._causal(hw_, L, cin, prod, self.out_rgb, 3, 2, stream=s)
                    return self.out_rgb[:npx * 3].view(T_, H_, W_, 3)
                self._causal(hw_, L, cin, prod, self.out_f, 32, F32, stream=s)
                return self.out_f[:npx * 32].view(T_, H_, W_, 32)
        raise ConfigError("VAE program has no head")

    def _mid_attention(self, name, L, C, s):
        """x += proj(softmax(q k^T / sqrt(C)) v) per frame, q/k/v = qkv(rms(x)) (1x1 convs as
        GEMMs over the pixels): scores as an fp32 GEMM per frame, a row softmax to bf16 P, V
        transposed into the K-major operand of the P.V GEMM, and the projection added into the
        fp32 residual stream by the GEMM's residual epilogue. Split decode: each rank's query rows
        attend to every rank's keys (all_gather_rows of K|V)."""
        T_, H_, W_ = L["T"], L["H"], L["W"]
        HWl, npx = H_ * W_, T_ * H_ * W_
        x, a = L["x"], self.attn
        u = L["xb"][:npx * C].view(npx, C)
        with ops._Prof("vae_norm", 0.0, float(npx) * C * 6, s):
            A.call("ftb_rmsnorm_silu_f32", A.ptr(x), npx, C, A.ptr(self.G[name + ".norm"]), 1e-12, 0, A.ptr(u),
                   A.stream_ptr(s))
        qkv = self.W[name + ".qkv"]
        q, kv = a["q"][:npx], a["kv"][:npx]
        ops.gemm(u, qkv.wt[:C], q, "bf16", bias=qkv.b[:C], stream=s, prof_kind="vae_attn")
        ops.gemm(u, qkv.wt[C:3 * C], kv, "bf16", bias=qkv.b[C:3 * C], stream=s, prof_kind="vae_attn")
        if self.split:
            h = sum(self.sizes)
            full = a["kv_full"]
            self.comm.all_gather_rows("vae_kv", full, kv.view(T_, H_, W_, 2 * C), self.sizes, s)
            kv_frames = full.view(T_, h * W_, 2 * C)
        else:
            kv_frames = kv.view(T_, HWl, 2 * C)
        HW = kv_frames.shape[1]
        vt, sc, pr = a["vt"][:, :HW], a["s"][:HWl, :HW], a["p"][:HWl, :HW]
        scale = 1.0 / float(np.sqrt(C))
        for t in range(T_):
            kt, vv = kv_frames[t][:, :C], kv_frames[t][:, C:]
            ops.transpose_bf16(vv, vt, stream=s)
            ops.gemm(q[t * HWl:(t + 1) * HWl], kt, sc, "f32", stream=s, prof_kind="vae_attn")
            ops.softmax_rows_bf16(sc, pr, scale, stream=s)
            ops.gemm(pr, vt, a["o"][t * HWl:(t + 1) * HWl], "bf16", stream=s, prof_kind="vae_attn")
        proj = self.W[name + ".proj"]
        ops.gemm(a["o"][:npx], proj.wt, x[:npx * C].view(npx, C), "resid_f32", bias=proj.b, stream=s,
                 prof_kind="vae_attn")

    def _next_norm(self, i, c):
        """Gain of the RMS norm that consumes op i's c-channel output (next resblock's norm1
        or the head norm) when it can ride op i's conv epilogue, else None."""
        if self.fuse_norm != "all" or c > 192 or i + 1 >= len(self.prog):
            return None
        op, name, cin, _ = self.prog[i + 1]
        if op == "res" and cin == c:
            return self.G[name + ".norm1"]
        if op == "head" and cin == c:
            return self.G["head.norm"]
        return None

    def _full_work(self, T, h, w, zc):
        buf = getattr(self, "_fw", None)
        n = (T + 2) * h * w * zc
        if buf is None or buf.numel() < n:
            buf = torch.empty(n, dtype=torch.bfloat16, device=self.dev)
            self._fw = buf
        return buf

    def decode_device(self, z, stream):
        """Codec interface of the streaming engine: device latents -> host frames. A split
        decoder gathers the slabs to rank 0, which returns the full frames; other ranks None."""
        with torch.cuda.stream(stream):
            out = self.decode_device_tensor(z.reshape(z.shape[0], self.cfg.z_dim, *z.shape[-2:]), stream,
                                            gather=True)
            if out is None:
                return None
            key = tuple(out.shape) + (out.dtype,)
            host = self._host.get(key)
            if host is None:
                host = torch.empty(out.shape, dtype=out.dtype).pin_memory()
                self._host[key] = host
            host.copy_(out, non_blocking=True)
        stream.synchronize()
        return host.numpy().copy()   # the pinned buffer is reused by the next chunk

    def decode_device_async(self, z, stream, slot=0, gather=False):
        """decode_device without the host wait: decode + D2H into pinned buffer `slot` are
        enqueued on `stream`; returns (pinned host tensor, event recorded after the copy).
        Two slots let chunk c's frames land while chunk c+1 is being enqueued. gather=True:
        split decoders collect the frames on rank 0 (other ranks get (None, None))."""
        with torch.cuda.stream(stream):
            out = self.decode_device_tensor(z.reshape(z.shape[0], self.cfg.z_dim, *z.shape[-2:]), stream,
                                            gather=gather)
            if out is None:
                return None, None
            key = tuple(out.shape) + (out.dtype, int(slot))
            host = self._host.get(key)
            if host is None:
                host = torch.empty(out.shape, dtype=out.dtype).pin_memory()
                self._host[key] = host
            host.copy_(out, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        return host, ev

    def encode(self, frames):  # pragma: no cover - encoder is out of scope
        raise ConfigError("the VAE encoder is out of scope; pass reference_latent to start_stream")
