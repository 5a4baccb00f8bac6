"""Denoiser API mirror (reference `pkg/src/ftlk/net.py`): NetConfig, ParamStore,
sinusoid_features, Denoiser.forward / as_denoise_fn — executed on the B200.

`ParamStore` keeps the reference's host float64 parameter table (same names,
same (in, out) layout, same seeded init `net.py:99-112`, same checksum), so a
reference checkpoint or init maps 1:1. `Denoiser.forward(store, comp)` uploads
the store once (bf16 W^T, fp32 vectors; cached per store) and runs the whole
forward in sm_100a kernels; the returned x0 prediction is float64 on the host
like the reference's. Backward / optimisers are training-only and out of scope.
"""

import hashlib
import weakref

import numpy as np
import torch

from .config import NetConfig, param_shapes
from .diffusion import CompositeInput
from .errors import ConfigError
from .model import DeviceDenoiser, DeviceWeights, sinusoid
from .seeding import INIT, rng_for

sinusoid_features = sinusoid


class ParamStore:
    """Named float64 parameter arrays (reference layout)."""

    def __init__(self, params: dict):
        self.params = {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in params.items()}

    @classmethod
    def zeros(cls, cfg: NetConfig):
        return cls({name: np.zeros(shape) for name, shape in param_shapes(cfg)})

    @classmethod
    def init(cls, cfg: NetConfig, seed: int):
        """Gains 1, biases 0, matrices N(0,1)/sqrt(fan_in) in table order from
        rng_for(seed, INIT) (net.py:99-112). Extension `.mod` tables use
        1/sqrt(model_dim)."""
        rng = rng_for(seed, INIT)
        params = {}
        for name, shape in param_shapes(cfg):
            if name.endswith(".g"):
                params[name] = np.ones(shape)
            elif name.endswith(".b") or len(shape) == 1:
                params[name] = np.zeros(shape)
            elif name.endswith(".mod"):
                params[name] = rng.standard_normal(shape) / np.sqrt(shape[-1])
            else:
                params[name] = rng.standard_normal(shape) / np.sqrt(shape[0])
        return cls(params)

    def names(self):
        return list(self.params.keys())

    @property
    def n_params(self):
        return sum(v.size for v in self.params.values())

    def checksum(self):
        h = hashlib.sha256()
        for name, v in self.params.items():
            h.update(name.encode())
            h.update(np.ascontiguousarray(v).tobytes())
        return h.hexdigest()

    def clone(self):
        return ParamStore({k: v.copy() for k, v in self.params.items()})

    def bf16_rounded(self):
        """Copy with every tensor rounded to bf16 and back (the values the
        device actually uses; feeding these to an fp64 oracle isolates kernel
        arithmetic error from weight quantisation)."""
        out = {}
        for k, v in self.params.items():
            out[k] = torch.from_numpy(v).to(torch.bfloat16).to(torch.float64).numpy()
        return ParamStore(out)


class _DeviceRunner:
    """Device weights of one ParamStore + per-geometry DeviceDenoiser cache. With a
    communicator (dist.py) the denoisers run Ulysses sequence parallel over its ranks; every
    rank holds the same runner (replicated weights and sampler state)."""

    def __init__(self, cfg, store, device, comm=None):
        self.cfg = cfg
        self.device = torch.device(device)
        self.comm = comm
        if isinstance(store, DeviceWeights):   # already resident (checkpoint.load_device_weights, synthetic)
            if store.cfg != cfg:
                raise ConfigError("device weights were built for a different NetConfig")
            self.weights = store
            self.device = store.device
        else:
            self.weights = DeviceWeights.from_host(cfg, store.params, self.device)
        self._geo = {}
        self.stream = None

    def denoiser(self, lc, lm, hw):
        key = (lc, lm, tuple(hw))
        d = self._geo.get(key)
        if d is None:
            d = DeviceDenoiser(self.weights, lc, lm, hw, stream=self.stream, comm=self.comm)
            self._geo[key] = d
        return d

    def _geometry(self, latents_shape, lc, lm):
        hw = latents_shape[2:] if self.cfg.mode == "wan" else (1, 1)
        if self.cfg.mode == "wan" and len(hw) != 2:
            raise ConfigError("wan mode latents must be (frames, D, H, W)")
        return self.denoiser(lc, lm, hw)

    def _dev(self, a, shape):
        return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32).reshape(shape)).to(self.device)

    def forward_host(self, comp: CompositeInput):
        cfg = self.cfg
        lc, lm = comp.chunk_len, comp.motion_len
        if comp.latent_dim != cfg.latent_dim:
            raise ConfigError("composite latent dim %d != net latent dim %d" % (comp.latent_dim, cfg.latent_dim))
        d = self._geometry(comp.z_noise.shape, lc, lm)
        fshape = (d.cfg.latent_dim, d.H, d.W)
        mask_ok = comp.z_mask[0] == 1.0 and not np.any(comp.z_mask[1:])
        cond_ok = np.array_equal(comp.z_cond[0], comp.reference) and not np.any(comp.z_cond[1:])
        d.prepare_cond(comp.signal, comp.reference)
        fv = d.frame_vectors(comp.frame_t)
        if mask_ok and cond_ok:   # Eq.1 assembled on device from motion / z / reference
            motion = self._dev(comp.z_noise[:lm], (lm,) + fshape) if lm else None
            z = self._dev(comp.z_noise[lm:], (lc - lm,) + fshape)
            ref = self._dev(comp.reference, fshape)
            x0t = d.step(motion, z, ref, fv)
        else:                     # any other composite (own mask / conditioning rows): upload it whole
            st = self._dev(comp.stacked(), (lc, 2 * d.cfg.latent_dim + 1, d.H, d.W))
            x0t = d.step(None, None, None, fv, stacked=st)
        out = d.tokens_to_frames(x0t).to(torch.float64).cpu().numpy()
        return out.reshape(comp.z_noise.shape)

    def sample_host(self, plan, motion, reference, signal, z, trace=None):
        lm = motion.shape[0]
        lc = lm + z.shape[0]
        d = self._geometry((lc,) + reference.shape[:1] + tuple(reference.shape[1:]), lc, lm)
        fshape = (d.cfg.latent_dim, d.H, d.W)
        md = self._dev(motion, (lm,) + fshape) if lm else None
        zd = self._dev(z, (lc - lm,) + fshape)
        rd = self._dev(reference, fshape)
        x0 = torch.empty((lc - lm,) + fshape, dtype=torch.float32, device=self.device)
        d.prepare_cond(signal, reference)
        dtrace = [] if trace is not None else None
        d.sample(md, rd, zd, plan, x0, trace=dtrace)
        if trace is not None:
            for t, zz, xx in dtrace:
                trace.append((t, zz.double().cpu().numpy().reshape(z.shape), xx.double().cpu().numpy().reshape(z.shape)))
        x0h = x0.double().cpu().numpy().reshape(z.shape)
        return np.concatenate([motion, x0h], axis=0)


_RUNNERS = weakref.WeakKeyDictionary()


def device_runner(cfg, store, device="cuda", comm=None):
    per = _RUNNERS.setdefault(store, {})
    key = (cfg, str(device), id(comm))
    r = per.get(key)
    if r is None:
        r = _DeviceRunner(cfg, store, device, comm)
        per[key] = r
    return r


class Denoiser:
    """Stateless evaluator over a ParamStore (net.py:209-375), device-backed."""

    def __init__(self, cfg: NetConfig, device="cuda", comm=None):
        self.cfg = cfg
        self.device = device
        self.comm = comm   # optional Ulysses communicator (every rank calls with the same inputs)

    def init_params(self, seed: int) -> ParamStore:
        return ParamStore.init(self.cfg, seed)

    def forward(self, params_store: ParamStore, comp: CompositeInput) -> np.ndarray:
        return device_runner(self.cfg, params_store, self.device, self.comm).forward_host(comp)

    def as_denoise_fn(self, params_store: ParamStore):
        runner = device_runner(self.cfg, params_store, self.device, self.comm)

        def fn(comp: CompositeInput) -> np.ndarray:
            return runner.forward_host(comp)

        fn._ftb_device = runner
        return fn
