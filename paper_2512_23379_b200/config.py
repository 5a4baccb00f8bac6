"""Model / sampler / stream configuration mirrors.

Field names and validation follow the reference so a reference config maps
1:1 onto these dataclasses:

* `NetConfig`    <- `pkg/src/ftlk/net.py:27-53`   (+ B200 extension fields)
* `NoiseSchedule`, `SamplerPlan` <- `pkg/src/ftlk/diffusion.py:16-58`
* `StreamConfig` <- `pkg/src/ftlk/streaming.py:43-69`

Extension (not in the reference): `mode="wan"` selects the Wan-shaped DiT
(spatial 2x2 patch tokens, 3D RoPE, AdaLN modulation + gating, multi-token
audio conditioning). `mode="ftlk"` (default) is the reference-exact model.
"""

from dataclasses import dataclass, field

from .errors import ConfigError

MODES = ("ftlk", "wan")
PACING_MODES = ("realtime", "unpaced")


@dataclass(frozen=True)
class NetConfig:
    model_dim: int = 32
    layers: int = 2
    heads: int = 2
    ff_dim: int = 64
    latent_dim: int = 8
    # ---- B200 extension (defaults reproduce the reference exactly) ----
    mode: str = "ftlk"
    patch: tuple = (1, 2, 2)        # wan: (t, h, w) patch of the latent grid; t must be 1
    audio_dim: int = 1              # wan: per-token driving feature width
    audio_tokens: int = 1           # wan: driving tokens per latent frame
    rope_theta: float = 10000.0     # wan: 3D RoPE base

    def validate(self) -> list:
        problems = []
        for name in ("model_dim", "layers", "heads", "ff_dim", "latent_dim"):
            if getattr(self, name) < 1:
                problems.append(f"net.{name} must be >= 1")
        if self.model_dim % max(self.heads, 1) != 0:
            problems.append("net.model_dim must be divisible by net.heads")
        if self.model_dim % 2 != 0:
            problems.append("net.model_dim must be even (sinusoidal embeddings)")
        if self.mode not in MODES:
            problems.append(f"net.mode must be one of {MODES}")
        if self.mode == "wan":
            if len(tuple(self.patch)) != 3 or tuple(self.patch)[0] != 1:
                problems.append("net.patch must be (1, ph, pw)")
            if self.audio_dim < 1 or self.audio_tokens < 1:
                problems.append("net.audio_dim and net.audio_tokens must be >= 1")
            hd = self.model_dim // max(self.heads, 1)
            if hd % 2 != 0 or hd < 8:
                problems.append("net head_dim must be even and >= 8 for 3D RoPE")
        return problems

    def __post_init__(self):
        object.__setattr__(self, "patch", tuple(int(p) for p in self.patch))
        problems = self.validate()
        if problems:
            raise ConfigError(problems)

    @property
    def input_channels(self) -> int:
        return 2 * self.latent_dim + 1

    @property
    def head_dim(self) -> int:
        return self.model_dim // self.heads

    @property
    def patch_area(self) -> int:
        return self.patch[1] * self.patch[2] if self.mode == "wan" else 1

    @property
    def in_features(self) -> int:
        """Per-token input width of the in-projection."""
        return self.input_channels * self.patch_area

    @property
    def out_features(self) -> int:
        return self.latent_dim * self.patch_area

    @property
    def cond_dim(self) -> int:
        return self.audio_dim if self.mode == "wan" else 1


def param_shapes(cfg: NetConfig):
    """Ordered (name, shape) list. ftlk mode is the reference layout
    (`pkg/src/ftlk/net.py:56-85`, weights stored (in, out)); wan mode adds the
    AdaLN projections and drops the affine pre-norms it replaces."""
    m, ff, d = cfg.model_dim, cfg.ff_dim, cfg.latent_dim
    wan = cfg.mode == "wan"
    shapes = [
        ("in.w", (cfg.in_features, m)), ("in.b", (m,)),
        ("time.w", (m, m)), ("time.b", (m,)),
    ]
    if wan:
        shapes += [("tproj.w", (m, 6 * m)), ("tproj.b", (6 * m,))]
    shapes += [
        ("sig.w", (cfg.cond_dim, m)), ("sig.b", (m,)),
        ("ref.w", (d, m)), ("ref.b", (m,)),
    ]
    for i in range(cfg.layers):
        p = f"layers.{i}."
        block = []
        if wan:
            block.append((p + "mod", (6, m)))
        else:
            block += [(p + "ln1.g", (m,)), (p + "ln1.b", (m,))]
        block += [(p + "self.wq", (m, m)), (p + "self.wk", (m, m)),
                  (p + "self.wv", (m, m)), (p + "self.wo", (m, m)),
                  (p + "ln2.g", (m,)), (p + "ln2.b", (m,)),
                  (p + "cross.wq", (m, m)), (p + "cross.wk", (m, m)),
                  (p + "cross.wv", (m, m)), (p + "cross.wo", (m, m))]
        if not wan:
            block += [(p + "ln3.g", (m,)), (p + "ln3.b", (m,))]
        block += [(p + "ffn.w1", (m, ff)), (p + "ffn.b1", (ff,)),
                  (p + "ffn.w2", (ff, m)), (p + "ffn.b2", (m,))]
        shapes += block
    if wan:
        shapes += [("final.mod", (2, m))]
    else:
        shapes += [("final.g", (m,)), ("final.b", (m,))]
    shapes += [("out.w", (m, cfg.out_features)), ("out.b", (cfg.out_features,))]
    return shapes


def n_params(cfg: NetConfig) -> int:
    total = 0
    for _, shape in param_shapes(cfg):
        n = 1
        for s in shape:
            n *= s
        total += n
    return total


@dataclass(frozen=True)
class NoiseSchedule:
    """Rectified-linear schedule alpha = 1 - t, sigma = t (diffusion.py:16-28)."""

    kind: str = "rectified_linear"

    def __post_init__(self):
        if self.kind != "rectified_linear":
            raise ConfigError(f"unknown schedule kind: {self.kind!r}")

    def alpha(self, t) -> float:
        return 1.0 - float(t)

    def sigma(self, t) -> float:
        return float(t) + 0.0


@dataclass(frozen=True)
class SamplerPlan:
    """Few-step ladder, first entry pinned at t=1 (diffusion.py:31-58)."""

    steps: int = 4
    timesteps: tuple = (1.0, 0.75, 0.5, 0.25)
    schedule: NoiseSchedule = field(default_factory=NoiseSchedule)

    def validate(self) -> list:
        ts = tuple(self.timesteps)
        problems = []
        if self.steps < 1:
            problems.append("sampler.steps must be >= 1")
        if len(ts) != self.steps:
            problems.append("sampler.timesteps length must equal steps")
        if ts and ts[0] != 1.0:
            problems.append("sampler.timesteps must start at exactly 1.0")
        if any(later >= earlier for earlier, later in zip(ts, ts[1:])):
            problems.append("sampler.timesteps must be strictly decreasing")
        if ts and (ts[-1] < 0.0 or any(t <= 0.0 for t in ts[:-1])):
            problems.append("sampler.timesteps must stay in (0, 1] (last may be 0)")
        return problems

    def __post_init__(self):
        object.__setattr__(self, "timesteps", tuple(float(t) for t in self.timesteps))
        problems = self.validate()
        if problems:
            raise ConfigError(problems)

    def ddim_coefficients(self):
        """Per step i (except the last): z' = ca*x0 + cz*z with
        eps = (z - a_i x0)/s_i, z' = a_{i+1} x0 + s_{i+1} eps
        => ca = a_{i+1} - s_{i+1} a_i / s_i, cz = s_{i+1} / s_i."""
        sch = self.schedule
        out = []
        for i in range(self.steps - 1):
            t, tn = self.timesteps[i], self.timesteps[i + 1]
            a, s = sch.alpha(t), sch.sigma(t)
            an, sn = sch.alpha(tn), sch.sigma(tn)
            out.append((a, s, an, sn))
        return out


@dataclass(frozen=True)
class StreamConfig:
    chunk_len: int = 9
    motion_len: int = 2
    target_fps: float = 25.0
    sampler: SamplerPlan = field(default_factory=SamplerPlan)
    seed: int = 0
    pacing: str = "unpaced"

    def validate(self) -> list:
        problems = []
        if not (0 <= self.motion_len < self.chunk_len):
            problems.append("stream.motion_len must satisfy 0 <= L_m < L_c")
        if self.target_fps <= 0:
            problems.append("stream.target_fps must be > 0")
        if self.pacing not in PACING_MODES:
            problems.append(f"stream.pacing must be one of {PACING_MODES}")
        return problems

    def __post_init__(self):
        problems = self.validate()
        if problems:
            raise ConfigError(problems)

    @property
    def stride(self) -> int:
        return self.chunk_len - self.motion_len


# Named shapes used by tests and the bench (BASELINE.json configs).
TINY = NetConfig()                                               # C1: reference default
WAN_1_3B = NetConfig(model_dim=1536, layers=30, heads=12, ff_dim=8960, latent_dim=16,
                     mode="wan", patch=(1, 2, 2), audio_dim=768, audio_tokens=4)
WAN_14B = NetConfig(model_dim=5120, layers=40, heads=40, ff_dim=13824, latent_dim=16,
                    mode="wan", patch=(1, 2, 2), audio_dim=768, audio_tokens=4)

# Aspect-ratio buckets (pixel H, W); latent grid = /8, tokens = /16.
BUCKETS = {
    "landscape_416x720": (416, 720),
    "portrait_720x416": (720, 416),
    "landscape_480x832": (480, 832),
    "portrait_832x480": (832, 480),
    "square_512x512": (512, 512),
}
