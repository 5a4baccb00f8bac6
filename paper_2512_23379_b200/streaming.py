"""Chunked streaming engine on the B200 (reference `pkg/src/ftlk/streaming.py`).

Same public surface as the reference: `StreamConfig`, `start_stream`,
`StreamSession.push_signal / next_frames / stats / persistent_state_nbytes /
close`, `EmittedFrame`, `StreamStats`, plus the synchronous twin `generate`
(reference `metrics.rollout_stream`, metrics.py:128-149).

Geometry is the reference's, bit-exact (streaming.py:246-306):
  chunk c is ready once (c+1)*S driving samples arrived (S = L_c - L_m);
  window = samples[c*S - L_m, c*S - L_m + L_c), indices < 0 read 0.0;
  pending samples below (c+1)*S - L_m are pruned;
  noise = rng_for(seed, STREAM_NOISE, c) drawn on the host;
  motion <- last L_m latent frames of [motion; x0]; cold start = L_m copies
  of the encoded reference; emitted frame index = c * frames_per_chunk + j.

Execution: three host threads as in the reference, but the denoise stage
runs the whole 4-step ladder on a dedicated CUDA stream (device-resident
weights, motion cache and sampler state) and hands the chunk's target latents
to the decode stage through a CUDA event without waiting for them (the host
enqueues chunk n+1 while chunk n runs); the decode stage decodes on its own
stream (orthogonal codec or the causal VAE), copies frames to pinned host
memory and emits them, so decoding chunk n overlaps denoising chunk n+1.

Multi-GPU (north star "8xB200"): with `comm` (dist.py) every rank
runs the same session. Rank 0 owns the input: its ingest thread broadcasts
each ready chunk (index, driving window) to the other ranks over a host
channel, so every rank draws the same noise and keeps the same (replicated)
sampler state; the DiT step runs Ulysses sequence parallel over the ranks; a
spatially split VAE (built on `comm.channel("vae")`) decodes one row slab per
rank and gathers the frames into rank 0, which alone emits them.
"""

import collections
import queue
import sys
import threading
import time
import types
from dataclasses import dataclass

import numpy as np
import torch

from .config import PACING_MODES, SamplerPlan, StreamConfig  # noqa: F401
from . import ops
from .errors import ConfigError, NumericError
from .net import device_runner
from .seeding import chunk_noise

_RECENT = 64
_CYCLE_KEYS = ("signal_ms", "denoise_ms", "decode_ms", "motion_encode_ms", "misc_ms")


@dataclass
class StreamStats:
    startup_ms: float
    fps: float
    frames_emitted: int
    chunks_emitted: int
    generate_ms: float
    cycle: dict


@dataclass
class EmittedFrame:
    index: int
    chunk: int
    state: np.ndarray


def chunk_window(get, c, chunk_len, motion_len):
    """Indices and values of chunk c's driving window (streaming.py:262-264)."""
    stride = chunk_len - motion_len
    lo = c * stride - motion_len
    idx = list(range(lo, lo + chunk_len))
    return idx, [get(j) if j >= 0 else None for j in idx]


class DeviceStreamer:
    """Device state of one stream: denoiser at the stream geometry, motion
    cache, sampler state, and the codec. Used by StreamSession and generate()."""

    def __init__(self, runner, cfg: StreamConfig, codec, reference_latent, latent_hw=(1, 1), use_graph=True):
        self.runner, self.scfg, self.codec = runner, cfg, codec
        self.ncfg = runner.cfg
        self.dev = runner.device
        self.d = runner.denoiser(cfg.chunk_len, cfg.motion_len, latent_hw)
        d = self.d
        self.fshape = (self.ncfg.latent_dim, d.H, d.W)
        self.ref_host = np.asarray(reference_latent, dtype=np.float64).reshape(
            self.fshape if self.ncfg.mode == "wan" else (self.ncfg.latent_dim,))
        self.ref = torch.as_tensor(self.ref_host.reshape(self.fshape), dtype=torch.float32).to(self.dev)
        lm = cfg.motion_len
        self.motion = self.ref.unsqueeze(0).repeat(lm, 1, 1, 1).contiguous() if lm else None
        nt = cfg.stride
        self.z = torch.empty((nt,) + self.fshape, dtype=torch.float32, device=self.dev)
        self.noise_host = [torch.empty((nt,) + self.fshape, dtype=torch.float32).pin_memory() for _ in range(2)]
        self.x0_static = torch.empty((nt,) + self.fshape, dtype=torch.float32, device=self.dev)
        self.slots = [torch.empty((nt,) + self.fshape, dtype=torch.float32, device=self.dev) for _ in range(4)]
        self.slot = 0
        # per-chunk non-finite count of the target latents (device, inside the captured chunk)
        # and one pinned host copy per output slot, read by whoever waits for that chunk
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.nonfinite_host = [torch.zeros(1, dtype=torch.int32).pin_memory() for _ in range(4)]
        self.last_slot = 0
        self._k = 0
        self._h2d_ev = [None, None]
        self.use_graph = use_graph and (self.d.comm.world == 1 or getattr(self.d.comm, "capturable", False))
        self.graph = None
        self.graph_launches = 0
        self._eager_runs = 0

    def reset(self):
        lm = self.scfg.motion_len
        if lm:
            self.motion.copy_(self.ref.unsqueeze(0).expand(lm, *self.fshape))

    def _device_chunk(self):
        """All device work of one chunk after the H2D of its inputs: cond tokens and
        cross K/V, the 4-step ladder, the motion-cache update. CUDA-graph capturable."""
        cfg = self.scfg
        nt, lm = cfg.stride, cfg.motion_len
        self.d.upload_cond()
        self.d.sample(self.motion, self.ref, self.z, cfg.sampler, self.x0_static)
        ops.count_nonfinite(self.x0_static, self.nonfinite, stream=self.d.stream)
        if lm:
            if lm <= nt:
                self.motion.copy_(self.x0_static[nt - lm:])
            else:  # carried rows still include older motion rows
                keep = lm - nt
                self.motion.copy_(torch.cat([self.motion[lm - keep:], self.x0_static], 0))

    def _capture(self):
        """Capture _device_chunk once (after an eager warm-up filled the per-ladder
        caches); later chunks replay it: one launch instead of ~450 per step."""
        s = torch.cuda.Stream(device=self.dev)
        s.wait_stream(torch.cuda.current_stream())
        keep = self.d.stream
        self.d.stream = None
        g = torch.cuda.CUDAGraph()
        from . import _capi
        n0 = _capi.LAUNCHES[0]
        try:
            # thread_local: the engine's ingest / decode threads keep issuing their own CUDA work
            # (H2D staging, decode) while the denoise thread captures; only this thread's
            # capture-unsafe calls are errors
            with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
                self._device_chunk()
        finally:
            self.d.stream = keep
        self.graph_launches = _capi.LAUNCHES[0] - n0   # kernels per replay (bench gpu_launches)
        torch.cuda.current_stream().wait_stream(s)
        self.graph = g

    def run_resident(self, z_dev, cond_in_dev):
        """Chunk with inputs already in HBM (benchmark `value`): D2D into the static
        input buffers, then the captured graph (or the eager path before capture)."""
        self.z.copy_(z_dev)
        self.d.buf["cond_in"].copy_(cond_in_dev)
        if self.graph is not None:
            self.graph.replay()
        else:
            self._device_chunk()
            self._eager_runs += 1
            if self.use_graph and self._eager_runs == 1:
                self._capture()
        return self.x0_static

    def denoise_chunk(self, c, window, noise=None):
        with ops.nvtx("denoise chunk %d" % c):
            return self._denoise_chunk(c, window, noise)

    def _denoise_chunk(self, c, window, noise=None):
        """Runs chunk c on the current stream; returns the device x0 slot
        (targets). `noise` (host f64) defaults to the reference draw. Inputs are
        staged in pinned memory (double-buffered) and copied H2D in stream order."""
        cfg = self.scfg
        nt = cfg.stride
        if noise is None:
            noise = chunk_noise(cfg.seed, c, (nt,) + self.ref_host.shape)
        k = self._k
        self._k ^= 1
        if self._h2d_ev[k] is not None:
            self._h2d_ev[k].synchronize()   # staging buffer k no longer read by chunk c-2's copy
        self.noise_host[k].copy_(torch.from_numpy(np.asarray(noise, dtype=np.float32).reshape(self.fshape[:0] + (
            nt,) + self.fshape)))
        self.d.stage_cond(window, self.ref_host, k)
        self.z.copy_(self.noise_host[k], non_blocking=True)
        self.d.copy_cond_in(k)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self._h2d_ev[k] = ev
        if self.graph is not None:
            self.graph.replay()
        else:
            self._device_chunk()
            self._eager_runs += 1
            if self.use_graph and self._eager_runs == 1:
                self._capture()
        x0 = self.slots[self.slot]
        self.nonfinite_host[self.slot].copy_(self.nonfinite, non_blocking=True)
        self.last_slot = self.slot
        self.slot = (self.slot + 1) % len(self.slots)
        x0.copy_(self.x0_static)
        return x0

    def check_finite(self, c, slot):
        """NumericError (reference errors.py:17-18) when chunk c's target latents held a NaN/Inf.
        Call after the chunk's work is known complete (the caller has synchronised with it)."""
        n = int(self.nonfinite_host[slot].item())
        if n:
            raise NumericError("chunk %d: %d non-finite target latents" % (c, n))


class StreamSession:
    """One live stream; command it from a single controller thread."""

    def __init__(self, store, net_cfg, codec, reference_frame, cfg: StreamConfig, *, device="cuda",
                 reference_latent=None, latent_hw=(1, 1), comm=None):
        self.cfg = cfg
        self.codec = codec
        self._rank = comm.rank if comm is not None else 0
        self._world = comm.world if comm is not None else 1
        ccomm = getattr(codec, "comm", None)
        if ccomm is not None and ccomm.world not in (1, self._world):
            raise ConfigError("the decoder's communicator spans %d ranks, the session %d" % (ccomm.world,
                                                                                          self._world))
        # rank 0 broadcasts every ready chunk's window to the followers (collective: created here)
        self._host = comm.host_channel("ingest") if self._world > 1 else None
        runner = device_runner(net_cfg, store, device, comm)
        if reference_latent is None:
            reference_frame = np.asarray(reference_frame, dtype=np.float64)
            if net_cfg.mode == "ftlk" and reference_frame.shape != (net_cfg.latent_dim,):
                raise ConfigError("reference frame dimension does not match the net")
            reference_latent = codec.encode(reference_frame[None])[0]
        self._reference = np.asarray(reference_latent, dtype=np.float64)
        self._ds = DeviceStreamer(runner, cfg, codec, self._reference, latent_hw)
        self._sample_is_array = net_cfg.mode == "wan"
        self._pending = {}
        self._next_sample = 0
        self._next_window = 0
        self._inbox = queue.Queue()
        self._to_denoise = queue.Queue(maxsize=2)
        self._to_decode = queue.Queue(maxsize=2)
        self._out = collections.deque()
        self._out_cond = threading.Condition()
        self._lock = threading.Lock()
        self._closed = threading.Event()
        self._error = None
        self._t_start = time.perf_counter()
        self._startup_ms = -1.0
        self._last_emit_t = -1.0
        self._cycle_ring = np.zeros(_RECENT)
        self._cycle_count = 0
        self._frames_emitted = 0
        self._chunks_emitted = 0
        self._last_generate_ms = 0.0
        self._last_cycle = {k: 0.0 for k in _CYCLE_KEYS}
        self._denoise_stream = torch.cuda.Stream(device=runner.device)
        self._decode_stream = torch.cuda.Stream(device=runner.device)
        self._workers = [
            threading.Thread(target=self._ingest_loop if self._rank == 0 else self._follow_loop, daemon=True,
                             name="ftb-ingest"),
            threading.Thread(target=self._denoise_loop, daemon=True, name="ftb-denoise"),
            threading.Thread(target=self._decode_loop, daemon=True, name="ftb-decode"),
        ]
        for w in self._workers:
            w.start()

    # ---------------------------------------------------------------- controller API
    def push_signal(self, samples) -> int:
        if self._rank != 0:
            raise ConfigError("rank %d follows rank 0's chunk schedule: push the driving signal on rank 0"
                              % self._rank)
        if self._closed.is_set():
            raise ConfigError("session is closed")
        self._raise_pending_error()
        batch = []
        for i, v in samples:
            i = int(i)
            if i != self._next_sample:
                raise ConfigError("driving sample index %d out of order (expected %d)" % (i, self._next_sample))
            v = np.asarray(v, dtype=np.float64) if self._sample_is_array else float(v)
            if not np.all(np.isfinite(v)):
                raise ConfigError("driving sample %d is not finite" % i)
            batch.append((i, v))
            self._next_sample += 1
        self._inbox.put(batch)
        return len(batch)

    def next_frames(self, wait: bool = False, timeout: float = 0.05):
        self._raise_pending_error()
        with self._out_cond:
            if wait and not self._out and not self._closed.is_set():
                self._out_cond.wait(timeout)
            frames = list(self._out)
            self._out.clear()
        self._raise_pending_error()
        return frames, self.stats()

    def stats(self) -> StreamStats:
        with self._lock:
            n = min(self._cycle_count, _RECENT)
            mean_cycle = float(np.mean(self._cycle_ring[:n])) if n else 0.0
            fpc = self.frames_per_chunk
            fps = (fpc * 1000.0 / mean_cycle) if mean_cycle > 0 else 0.0
            return StreamStats(max(self._startup_ms, 0.0), fps, self._frames_emitted, self._chunks_emitted,
                               self._last_generate_ms, dict(self._last_cycle))

    @property
    def frames_per_chunk(self):
        return self.cfg.stride * getattr(self.codec, "frames_per_latent", 1)

    def persistent_state_nbytes(self) -> int:
        for _ in range(50):
            try:
                return _deep_nbytes(self.__dict__)
            except RuntimeError:
                time.sleep(0.002)
        return _deep_nbytes(self.__dict__)

    def close(self) -> None:
        if self._closed.is_set():
            return
        self._closed.set()
        self._inbox.put(None)
        with self._out_cond:
            self._out_cond.notify_all()
        for w in self._workers:
            w.join(timeout=10.0)

    # ---------------------------------------------------------------- workers
    def _fail(self, exc):
        self._error = exc
        self._closed.set()
        with self._out_cond:
            self._out_cond.notify_all()

    def _raise_pending_error(self):
        if self._error is not None:
            raise self._error

    def _ingest_loop(self):
        cfg = self.cfg
        received = 0
        zero = None
        try:
            while not self._closed.is_set():
                batch = self._inbox.get()
                if batch is None:
                    break
                t0 = time.perf_counter()
                for i, v in batch:
                    self._pending[i] = v
                    if zero is None:
                        zero = np.zeros_like(v) if isinstance(v, np.ndarray) else 0.0
                received += len(batch)
                signal_ms = (time.perf_counter() - t0) * 1000.0
                while received >= (self._next_window + 1) * cfg.stride:
                    c = self._next_window
                    t1 = time.perf_counter()
                    _, vals = chunk_window(lambda j: self._pending.get(j, zero), c, cfg.chunk_len, cfg.motion_len)
                    window = np.array([zero if v is None else v for v in vals], dtype=np.float64)
                    keep_from = (c + 1) * cfg.stride - cfg.motion_len
                    self._pending = {j: v for j, v in self._pending.items() if j >= keep_from}
                    self._next_window += 1
                    if self._host is not None:
                        self._host.host_broadcast((c, window))     # followers run the same chunk
                    noise = chunk_noise(cfg.seed, c, (cfg.stride,) + self._reference.shape)
                    signal_ms += (time.perf_counter() - t1) * 1000.0
                    t_origin = time.perf_counter() - signal_ms / 1000.0
                    self._to_denoise.put((c, window, noise, signal_ms, t_origin))
                    signal_ms = 0.0
        except Exception as exc:  # noqa: BLE001
            self._fail(exc)
        finally:
            if self._host is not None:
                try:
                    self._host.host_broadcast(None)                # end of stream for the followers
                except Exception as exc:  # noqa: BLE001
                    self._fail(exc)
            self._to_denoise.put(None)

    def _follow_loop(self):
        """Ranks > 0: the chunk schedule comes from rank 0 (same windows, same noise draw)."""
        cfg = self.cfg
        try:
            while True:
                item = self._host.host_broadcast(None)
                if item is None:
                    break
                t0 = time.perf_counter()
                c, window = item
                self._next_window = c + 1
                noise = chunk_noise(cfg.seed, c, (cfg.stride,) + self._reference.shape)
                self._to_denoise.put((c, window, noise, (time.perf_counter() - t0) * 1000.0, t0))
        except Exception as exc:  # noqa: BLE001
            self._fail(exc)
        finally:
            self._to_denoise.put(None)

    def _denoise_loop(self):
        try:
            with torch.cuda.device(self._ds.dev), torch.cuda.stream(self._denoise_stream):
                self._ds.d.stream = self._denoise_stream
                while True:
                    item = self._to_denoise.get()
                    if item is None:
                        break
                    c, window, noise, signal_ms, t_ready = item
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record(self._denoise_stream)
                    x0 = self._ds.denoise_chunk(c, window, noise)
                    slot = self._ds.last_slot
                    ev = torch.cuda.Event(enable_timing=True)
                    ev.record(self._denoise_stream)
                    # no host wait: the decode stage waits on `ev`, this thread enqueues chunk c+1
                    # (the 4-slot x0 ring and the 2-deep decode queue keep chunk c's slot alive)
                    self._to_decode.put((c, x0, (e0, ev, slot), signal_ms, 0.0, t_ready))
        except Exception as exc:  # noqa: BLE001
            self._fail(exc)
        finally:
            self._to_decode.put(None)

    def _decode_loop(self):
        cfg = self.cfg
        chunk_period = self.frames_per_chunk / cfg.target_fps
        next_due = None
        try:
            with torch.cuda.device(self._ds.dev), torch.cuda.stream(self._decode_stream):
                while True:
                    item = self._to_decode.get()
                    if item is None:
                        break
                    c, x0, (e0, ev, slot), signal_ms, motion_ms, t_ready = item
                    if cfg.pacing == "realtime":
                        now = time.perf_counter()
                        if next_due is None:
                            next_due = now
                        if next_due > now:
                            time.sleep(next_due - now)
                        next_due += chunk_period
                    self._decode_stream.wait_event(ev)
                    d0 = torch.cuda.Event(enable_timing=True)
                    d0.record(self._decode_stream)
                    with ops.nvtx("decode chunk %d" % c):
                        frames = self.codec.decode_device(x0, self._decode_stream)   # waits for the frames
                    d1 = torch.cuda.Event(enable_timing=True)
                    d1.record(self._decode_stream)
                    d1.synchronize()
                    self._ds.check_finite(c, slot)
                    denoise_ms = e0.elapsed_time(ev)
                    decode_ms = d0.elapsed_time(d1)
                    if self._rank != 0:
                        frames = None      # rank 0 emits (a split decoder gathered the frames there)
                    fpc = self.frames_per_chunk if frames is None else len(frames)
                    emitted = [] if frames is None else [EmittedFrame(c * fpc + j, c, frames[j]) for j in range(fpc)]
                    t_emit = time.perf_counter()
                    total_ms = (t_emit - t_ready) * 1000.0
                    misc_ms = max(0.0, total_ms - signal_ms - denoise_ms - decode_ms - motion_ms)
                    with self._lock:
                        if self._startup_ms < 0:
                            self._startup_ms = (t_emit - self._t_start) * 1000.0
                        if self._last_emit_t >= 0:
                            self._cycle_ring[self._cycle_count % _RECENT] = (t_emit - self._last_emit_t) * 1000.0
                            self._cycle_count += 1
                        self._last_emit_t = t_emit
                        self._frames_emitted += len(emitted)
                        self._chunks_emitted += 1 if emitted else 0
                        self._last_generate_ms = denoise_ms + decode_ms
                        self._last_cycle = {"signal_ms": signal_ms, "denoise_ms": denoise_ms,
                                            "decode_ms": decode_ms, "motion_encode_ms": motion_ms,
                                            "misc_ms": misc_ms}
                    with self._out_cond:
                        self._out.extend(emitted)
                        self._out_cond.notify_all()
        except Exception as exc:  # noqa: BLE001
            self._fail(exc)


def start_stream(store, net_cfg, codec, reference_frame, cfg: StreamConfig, **kw) -> StreamSession:
    """streaming.py:359-361. `store`: the reference's ParamStore (uploaded once, cached per
    store) or device-resident weights (`model.DeviceWeights`, e.g. from
    `checkpoint.load_device_weights` — a 14B host fp64 store would need 105 GiB)."""
    return StreamSession(store, net_cfg, codec, reference_frame, cfg, **kw)


def generate(store, net_cfg, codec, reference_latent, signal, n_frames, *, cfg: StreamConfig = None,
             device="cuda", latent_hw=(1, 1), decode=True, motion_override=None, comm=None):
    """Synchronous chunked generation with the engine's exact geometry (the
    reference's `rollout_stream`, metrics.py:128-149). Returns
    (targets (n_frames_latent, ...), motions per chunk, decoded frames or None).
    `motion_override[c]` teacher-forces chunk c's motion rows (parity tests).
    With `comm` every rank calls it with the same arguments (Ulysses DiT, replicated
    sampler state); a split decoder returns the frames on rank 0 only."""
    cfg = cfg or StreamConfig()
    runner = device_runner(net_cfg, store, device, comm)
    ds = DeviceStreamer(runner, cfg, codec, reference_latent, latent_hw)
    stride = cfg.stride
    n_chunks = int(np.ceil(n_frames / stride))
    signal = np.asarray(signal, dtype=np.float64)
    zero = np.zeros(signal.shape[1:]) if signal.ndim > 1 else 0.0
    outs, motions, frames = [], [], []
    for c in range(n_chunks):
        _, vals = chunk_window(lambda j: signal[j] if j < len(signal) else zero, c, cfg.chunk_len, cfg.motion_len)
        window = np.array([zero if v is None else v for v in vals], dtype=np.float64)
        if motion_override is not None and cfg.motion_len:
            ds.motion.copy_(torch.as_tensor(np.asarray(motion_override[c], dtype=np.float32)).reshape(
                ds.motion.shape))
        motions.append(ds.motion.double().cpu().numpy().reshape((cfg.motion_len,) + ds.ref_host.shape)
                       if cfg.motion_len else np.zeros((0,) + ds.ref_host.shape))
        x0 = ds.denoise_chunk(c, window)
        outs.append(x0.double().cpu().numpy().reshape((stride,) + ds.ref_host.shape))
        ds.check_finite(c, ds.last_slot)
        if decode and codec is not None:
            fr = codec.decode_device(x0, torch.cuda.current_stream())
            if fr is not None:
                frames.append(fr)
    targets = np.concatenate(outs, axis=0)[:n_frames]
    fr = np.concatenate(frames, axis=0) if frames else None
    return targets, motions, fr


_SIZE_OPAQUE = (type, types.ModuleType, types.FunctionType, types.MethodType, types.BuiltinFunctionType,
                threading.Thread)


def _deep_nbytes(obj, seen=None):
    """Host-side deep size of the live session (streaming.py:93-120); device
    tensors count their storage bytes so device-state growth shows too."""
    if isinstance(obj, (int, float, complex, bool, str, bytes, type(None))):
        return sys.getsizeof(obj)
    if seen is None:
        seen = set()
    if id(obj) in seen:
        return 0
    seen.add(id(obj))
    if isinstance(obj, np.ndarray):
        return int(obj.nbytes) + sys.getsizeof(obj)
    if isinstance(obj, torch.Tensor):
        return int(obj.numel() * obj.element_size())
    if isinstance(obj, _SIZE_OPAQUE) or isinstance(obj, (torch.cuda.Stream, torch.cuda.Event)):
        return 0
    size = sys.getsizeof(obj)
    if isinstance(obj, dict):
        size += sum(_deep_nbytes(k, seen) + _deep_nbytes(v, seen) for k, v in obj.items())
    elif isinstance(obj, (list, tuple, set, frozenset, collections.deque)):
        size += sum(_deep_nbytes(x, seen) for x in obj)
    elif hasattr(obj, "__dict__"):
        size += _deep_nbytes(obj.__dict__, seen)
    return size
