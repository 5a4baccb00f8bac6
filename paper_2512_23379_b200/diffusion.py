"""Sampler-side API mirror: LatentChunk, CompositeInput, composite_from_state,
few_step_sample (reference `pkg/src/ftlk/diffusion.py:61-237`).

`few_step_sample(denoise_fn, plan, motion, reference, signal, rng)` keeps the
reference signature. When `denoise_fn` is a device denoiser closure (from
`Denoiser.as_denoise_fn`), the whole ladder runs on the B200: the initial
noise is drawn on the host from `rng` (bit-identical to the reference's draw,
diffusion.py:225), uploaded once, and every step - composite assembly, DiT
forward, x0 slice and DDIM update - stays on device. Any other callable gets
the reference's host recursion (so oracle denoisers plug in unchanged).
"""

from dataclasses import dataclass

import numpy as np

from .config import NoiseSchedule, SamplerPlan  # noqa: F401  (re-exported API)
from .errors import ConfigError


@dataclass(frozen=True)
class LatentChunk:
    latents: np.ndarray
    motion_len: int

    def __post_init__(self):
        object.__setattr__(self, "latents", np.asarray(self.latents, dtype=np.float64))
        if self.latents.ndim < 2:
            raise ConfigError("chunk latents must be (frames, ...)")
        if not (0 <= self.motion_len < len(self.latents)):
            raise ConfigError("motion_len must satisfy 0 <= L_m < L_c")

    @property
    def chunk_len(self):
        return len(self.latents)

    @property
    def motion(self):
        return self.latents[:self.motion_len]

    @property
    def targets(self):
        return self.latents[self.motion_len:]


@dataclass(frozen=True)
class CompositeInput:
    """Eq.1 input. ftlk: z_noise/z_cond (L_c, D), reference (D,), signal (L_c,).
    wan: z_noise/z_cond (L_c, D, H, W), reference (D, H, W),
    signal (L_c, audio_tokens, audio_dim) driving features."""

    z_noise: np.ndarray
    z_mask: np.ndarray
    z_cond: np.ndarray
    signal: np.ndarray
    reference: np.ndarray
    frame_t: np.ndarray
    motion_len: int

    def __post_init__(self):
        for name in ("z_noise", "z_mask", "z_cond", "signal", "reference", "frame_t"):
            object.__setattr__(self, name, np.asarray(getattr(self, name), dtype=np.float64))
        if self.z_noise.ndim < 2:
            raise ConfigError("z_noise must be (frames, dim, ...)")
        lc = self.z_noise.shape[0]
        if self.z_cond.shape != self.z_noise.shape:
            raise ConfigError("z_cond shape must match z_noise")
        if self.z_mask.shape != (lc,) or self.frame_t.shape != (lc,) or self.signal.shape[0] != lc:
            raise ConfigError("per-frame vectors must have length L_c")
        if self.reference.shape != self.z_noise.shape[1:]:
            raise ConfigError("reference must be a single latent frame")
        if not (0 <= self.motion_len < lc):
            raise ConfigError("motion_len must satisfy 0 <= L_m < L_c")

    @property
    def chunk_len(self):
        return self.z_noise.shape[0]

    @property
    def latent_dim(self):
        return self.z_noise.shape[1]

    def stacked(self):
        mask = np.broadcast_to(self.z_mask.reshape((-1, 1) + (1,) * (self.z_noise.ndim - 2)),
                               (self.chunk_len, 1) + self.z_noise.shape[2:])
        return np.concatenate([self.z_noise, mask, self.z_cond], axis=1)


def composite_from_state(motion, z_state, reference, signal, t, motion_t=None):
    z_state = np.asarray(z_state, dtype=np.float64)
    reference = np.asarray(reference, dtype=np.float64)
    if z_state.ndim == reference.ndim:
        z_state = z_state[None]
    motion = np.asarray(motion, dtype=np.float64)
    if motion.size == 0:
        motion = motion.reshape((0,) + z_state.shape[1:])
    if motion.ndim == reference.ndim:
        motion = motion[None]
    if motion.shape[1:] != z_state.shape[1:]:
        raise ConfigError("motion/target latent dims differ")
    lm = motion.shape[0]
    lc = lm + z_state.shape[0]
    signal = np.asarray(signal, dtype=np.float64)
    if signal.shape[0] != lc:
        raise ConfigError("signal must supply one entry per frame (%d)" % lc)
    z_noise = np.concatenate([motion, z_state], axis=0)
    z_mask = np.zeros(lc)
    z_mask[0] = 1.0
    z_cond = np.zeros_like(z_noise)
    z_cond[0] = reference
    frame_t = np.full(lc, float(t))
    frame_t[:lm] = 0.0 if motion_t is None else np.asarray(motion_t, dtype=np.float64)
    return CompositeInput(z_noise, z_mask, z_cond, signal, reference, frame_t, lm)


def few_step_sample(denoise_fn, plan: SamplerPlan, motion, reference, signal, rng, trace=None):
    reference = np.asarray(reference, dtype=np.float64)
    signal = np.asarray(signal, dtype=np.float64)
    motion = np.asarray(motion, dtype=np.float64)
    if motion.size == 0:
        motion = motion.reshape((0,) + reference.shape)
    if motion.ndim == reference.ndim:
        motion = motion[None]
    lm, lc = motion.shape[0], signal.shape[0]
    if lc - lm < 1:
        raise ConfigError("chunk must contain at least one target frame")
    z = rng.standard_normal((lc - lm,) + reference.shape)
    device = getattr(denoise_fn, "_ftb_device", None)
    if device is not None:
        lat = device.sample_host(plan, motion, reference, signal, z, trace=trace)
        return LatentChunk(lat, lm)
    sched = plan.schedule
    x0 = None
    for i, t in enumerate(plan.timesteps):
        pred = np.asarray(denoise_fn(composite_from_state(motion, z, reference, signal, t)))
        x0 = pred[lm:]
        if trace is not None:
            trace.append((float(t), z.copy(), x0.copy()))
        if i + 1 < plan.steps:
            tn = plan.timesteps[i + 1]
            eps = (z - sched.alpha(t) * x0) / sched.sigma(t)
            z = sched.alpha(tn) * x0 + sched.sigma(tn) * eps
    return LatentChunk(np.concatenate([motion, x0], axis=0), lm)
