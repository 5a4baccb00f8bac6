"""Benchmark: streaming FPS + per-chunk latency of the 14B-shape DiT hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--model 14b|1.3b|tiny] [--bucket landscape_416x720]

One bench step = one streaming chunk: the 4-step distilled DiT denoise of a
9-latent-frame chunk (2 motion + 7 target frames; L = 9 x 1170 = 10 530
tokens at 416x720) followed by the decode of its 7 target latents
(= 28 video frames). Metric: FPS = 28 * K / time, plus ms per chunk.

`value`  : device time (CUDA events, max over ranks) with all inputs already
           resident in HBM (noise, audio features pre-uploaded).
`e2e`    : the same chunks through the public engine API (`start_stream` ->
           `StreamSession.push_signal / next_frames`, the reference's streaming surface):
           host noise drawn with the reference's PCG64 stream, pinned H2D of noise +
           driving window, D2H of the decoded RGB8 frames every step, host wall time.
`roofline`: one extra instrumented chunk after the timed region, every GEMM
           launch bracketed by CUDA events on its stream: achieved =
           sum(2MNK) / sum(duration) vs MEASURED_PEAKS bf16_tflops_sustained.
`cpu_baseline`: the float64 oracle layer (oracle/cpu_baseline.py) on the
           host cores, extrapolated to the chunk (rank 0, N = 1 only).
Weights are random-init of the named shape, generated on device.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MODELS = {"14b": "WAN_14B", "1.3b": "WAN_1_3B", "tiny": "TINY"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="14b", choices=list(MODELS))
    ap.add_argument("--bucket", default="landscape_416x720")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--detail", action="store_true", help="per-shape kernel breakdown on stderr")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of the captured chunk graph")
    ap.add_argument("--overlap", action="store_true",
                    help="decode chunk c on a second stream while chunk c+1 denoises (the engine's thread "
                         "schedule); measured: same throughput on one B200, +105 ms chunk latency, so off by default")
    ap.add_argument("--comm", default="peer", choices=["peer", "nccl"],
                    help="N>1 Ulysses transport: exchanges fused into the producing kernels' epilogues over "
                         "NVLink peer memory (default), or NCCL all-to-all / all-gather collectives")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:  # noqa: BLE001
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw"

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        note = None
        if not self.lines:   # timed region shorter than the sampling period (tiny model): one
            try:             # sample right after it, while the clocks are still at the load state
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10)
                self.lines = [ln.strip() for ln in out.stdout.splitlines() if ln.strip()]
                note = "timed region shorter than the 200 ms sampling period: one sample right after it"
            except Exception:  # noqa: BLE001
                pass
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        res = {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
               "samples": len(sm)}
        if note:
            res["note"] = note
        return res


REF_KERNELS = ("dense_forward", "dense_backward", "gelu_forward", "gelu_backward", "layernorm_forward",
               "layernorm_backward", "mha_forward", "mha_backward")


def reference_tiny_chunks(n_chunks, backend):
    """C1: the reference itself (ftlk installed in baseline/_ref, the Cython extension built
    there), `metrics.rollout_stream` over `NetGenerator` (4-step ladder, NetConfig(), random
    init) unpaced, plus the orthogonal codec decode of every chunk's targets — the engine's
    per-chunk work (streaming.py:283-356). The kernel table is rebound to `backend` the way the
    reference's own benchmark does it (benchmarks/bench_backends.py:65-90). Returns per-chunk
    seconds (list) or raises ImportError when the reference is not installed."""
    refdir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(refdir, "ftlk")):
        raise ImportError("reference not installed in baseline/_ref")
    if refdir not in sys.path:
        sys.path.insert(0, refdir)
    import ftlk.backends as K
    from ftlk.diffusion import SamplerPlan
    from ftlk.metrics import NetGenerator, StreamContext, rollout_stream
    from ftlk.net import Denoiser, NetConfig
    from ftlk.world import Codec
    impl = K.get_backend(backend)
    saved = {n: getattr(K, n) for n in REF_KERNELS}
    for n in REF_KERNELS:
        setattr(K, n, getattr(impl, n))
    try:
        cfg = NetConfig()
        store = Denoiser(cfg).init_params(200)
        gen = NetGenerator(store, cfg, SamplerPlan())
        r = np.random.default_rng(0)
        codec = Codec(np.linalg.qr(r.standard_normal((cfg.latent_dim, cfg.latent_dim)))[0])
        times = []
        inner = gen.chunk

        def timed(ctx, c, motion, sig, rng):
            t0 = time.perf_counter()
            ch = inner(ctx, c, motion, sig, rng)
            codec.decode(ch.targets)
            times.append(time.perf_counter() - t0)
            return ch
        gen.chunk = timed
        ident = r.standard_normal(cfg.latent_dim)
        ctx = StreamContext(0, 0, ident, r.uniform(-1, 1, 7 * n_chunks), ident, codec.encode(ident))
        rollout_stream(gen, ctx, 7 * n_chunks)
        return times
    finally:
        for n, fn in saved.items():
            setattr(K, n, fn)


def reference_arm(args):
    """CPU reference path, rank 0 only (other ranks exit without work).
    tiny (C1): the reference itself, rollout_stream unpaced on both of its backends
    (python = NumPy, cython = its compiled extension), median chunk over >= 200 chunks per step.
    wan shapes: the oracle port of the reference's NumPy fp64 path, each step one layer on one
    latent frame of tokens extrapolated to the chunk (infeasible in full on a host)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2512_23379_b200 import config as C
    cfg = getattr(C, MODELS[args.model])
    if args.model == "tiny":
        per_step, det = [], {}
        for i in range(args.warmup + args.steps):
            t = reference_tiny_chunks(200, "cython")
            if i >= args.warmup:
                per_step.append(float(np.median(t)))
        det["cython_chunk_ms_median"] = 1000.0 * float(np.median(per_step))
        det["python_chunk_ms_median"] = 1000.0 * float(np.median(reference_tiny_chunks(200, "python")))
        chunk_s = float(np.median(per_step))
        fps = 7.0 / chunk_s
        cb = {"value": fps, "unit": "FPS", "cores": 1, "kind": "reference",
              "sample": "ftlk rollout_stream (NetGenerator, 4-step ladder) + Codec.decode, unpaced, cython "
                        "backend, median chunk of 200 per step (python backend: %.2f ms/chunk)" %
                        det["python_chunk_ms_median"]}
        line = {"metric": "streaming FPS (tiny ftlk-shape DiT, 4-step chunk, 7 frames/chunk)", "value": fps,
                "unit": "FPS", "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": chunk_s * 1000.0, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload_name(args), "model": args.model}, "cpu_baseline": cb,
                "e2e": {"value": fps, "unit": "FPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "detail": det}
        print(json.dumps(line), flush=True)
        return
    from oracle.cpu_baseline import extrapolated_chunk_seconds, make_layer
    H, W = C.BUCKETS[args.bucket]
    T = (H // 16) * (W // 16)
    L = 9 * T
    L_s = T       # one latent frame of tokens
    P = make_layer(cfg.model_dim, cfg.ff_dim)
    times, det = [], None
    for i in range(args.warmup + args.steps):
        chunk_s, det = extrapolated_chunk_seconds(cfg.model_dim, cfg.heads, cfg.ff_dim, cfg.layers, 4, L, L_s,
                                                  P=P, seed=i)
        if i >= args.warmup:
            times.append(chunk_s)
    chunk_s = float(np.median(times))
    fps = 28.0 / chunk_s
    cb = {"value": fps, "unit": "FPS", "cores": os.cpu_count(), "kind": "port",
          "sample": "one %s-width wan layer fwd (fp64 NumPy oracle) on one latent frame (%d of %d tokens), "
                    "self-attention core timed on %d of %d heads; extrapolated linear x L/Ls + attention x "
                    "(L/Ls)^2 to %d layers x 4 steps; DiT only" %
                    (args.model, L_s, L, det["attn_heads_timed"], cfg.heads, cfg.layers)}
    line = {"metric": "streaming FPS (%s-shape DiT, 4-step chunk, 28 frames/chunk)" % (
                {"14b": "14B", "1.3b": "1.3B"}[args.model]), "value": fps, "unit": "FPS",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": chunk_s * 1000.0, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": {"workload": workload_name(args), "model": args.model},
            "cpu_baseline": cb, "e2e": {"value": fps, "unit": "FPS", "h2d_bytes_per_step": 0,
                                         "d2h_bytes_per_step": 0}, "detail": det}
    print(json.dumps(line), flush=True)


def pick_comm(args, w, Lc, Lm, lat_hw, stream, dev):
    """Ulysses transport for N > 1. The fused peer transport is checked once against the
    NCCL collectives on one synthetic step (bitwise: same kernels, only store targets
    differ); a mismatch or an IPC failure selects NCCL and says why in config.comm."""
    import torch
    import torch.distributed as dist

    from paper_2512_23379_b200.dist import IpcPeerComm, TorchComm
    from paper_2512_23379_b200.model import DeviceDenoiser
    nccl = TorchComm()
    if args.comm == "nccl":
        return nccl, "nccl all_to_all/all_gather"
    try:
        peer = IpcPeerComm(dev)
        dp = DeviceDenoiser(w, Lc, Lm, lat_hw, stream=stream, comm=peer)
        dn = DeviceDenoiser(w, Lc, Lm, lat_hw, stream=stream, comm=nccl)
        rng = np.random.default_rng(3)
        cfg = w.cfg
        shp = (cfg.latent_dim, dp.H, dp.W)
        mo = torch.as_tensor(rng.standard_normal((Lm,) + shp), dtype=torch.float32, device=dev)
        z = torch.as_tensor(rng.standard_normal((Lc - Lm,) + shp), dtype=torch.float32, device=dev)
        ref = torch.as_tensor(rng.standard_normal(shp), dtype=torch.float32, device=dev)
        win = (rng.standard_normal((Lc, cfg.audio_tokens, cfg.audio_dim)) if cfg.mode == "wan"
               else rng.uniform(-1, 1, Lc))
        outs = []
        for dd in (dp, dn):
            dd.prepare_cond(win, ref.cpu().numpy())
            fv = dd.frame_vectors(np.where(np.arange(Lc) < Lm, 0.0, 1.0))
            outs.append(dd.step(mo, z, ref, fv).clone())
        torch.cuda.synchronize()
        same = torch.tensor([int(torch.equal(outs[0], outs[1]))], device=dev)
        dist.all_reduce(same, op=dist.ReduceOp.MIN)
        del dp, dn, outs
        if int(same.item()) != 1:
            return nccl, "nccl (peer transport check mismatched)"
        return peer, "peer: QKV/FMHA/out-proj epilogues store over NVLink + device flag barrier"
    except Exception as e:  # noqa: BLE001  (IPC unavailable on this node)
        return nccl, "nccl (peer transport unavailable: %s)" % str(e).splitlines()[0][:120]


def workload_name(args):
    if args.model == "tiny":   # C1: the reference's default NetConfig (9 tokens, no spatial grid)
        return "stream_chunk_tiny_ftlk_Lc9_Lm2_4step"
    return "stream_chunk_%s_%s_Lc9_Lm2_4step" % (args.model, args.bucket)


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2512_23379_b200 import _capi, ops
    from paper_2512_23379_b200 import config as C
    from paper_2512_23379_b200.model import DeviceDenoiser, DeviceWeights
    from paper_2512_23379_b200.seeding import chunk_noise

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FTB_EMULATE_RANKS=1 (tests only): every rank on GPU 0, gloo process group, peer transport
    # with host barriers — exercises the N>1 plumbing on a one-GPU box; the timing is meaningless
    emulate = world > 1 and os.environ.get("FTB_EMULATE_RANKS") == "1"
    if emulate:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if emulate:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], device="cpu" if emulate else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    cfg = getattr(C, MODELS[args.model])
    Hpx, Wpx = C.BUCKETS[args.bucket]
    lat_hw = (Hpx // 8, Wpx // 8) if cfg.mode == "wan" else (1, 1)
    scfg = C.StreamConfig()
    Lc, Lm, S = scfg.chunk_len, scfg.motion_len, scfg.stride
    frames_per_chunk = S * (4 if cfg.mode == "wan" else 1)

    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    w = DeviceWeights.synthetic(cfg, dev, seed=200)
    comm, comm_note = None, "none"
    if emulate:
        from paper_2512_23379_b200.dist import IpcPeerComm
        comm, comm_note = IpcPeerComm(dev, barrier_mode="host"), "peer (emulated ranks on one GPU, host barrier)"
    elif world > 1:
        # Ulysses sequence parallel: one chunk sharded over all ranks (strong scaling)
        comm, comm_note = pick_comm(args, w, Lc, Lm, lat_hw, stream, dev)
    d = DeviceDenoiser(w, Lc, Lm, lat_hw, stream=stream, comm=comm)
    fshape = (cfg.latent_dim,) + tuple(d.H and (d.H, d.W))
    A = cfg.audio_tokens if cfg.mode == "wan" else 1
    adim = cfg.audio_dim if cfg.mode == "wan" else 1
    rng = np.random.default_rng(7)            # every rank drives the same stream
    ref_host = rng.standard_normal(fshape)
    nsteps = args.warmup + args.steps
    windows = [rng.standard_normal((Lc, A, adim)) if cfg.mode == "wan" else rng.uniform(-1, 1, Lc)
               for _ in range(nsteps)]
    vae = None
    if cfg.mode == "wan" and not args.no_decode:   # N > 1: spatially split decode with halo exchange
        from paper_2512_23379_b200.vae import DeviceVAEDecoder, VAEConfig
        # the decode has its own channel (barrier flags / process group): in the engine it runs on
        # the decode stream concurrently with the denoise stream's Ulysses barriers
        vae = DeviceVAEDecoder(VAEConfig(z_dim=cfg.latent_dim), dev, params=None, seed=201, rgb8=True,
                               comm=comm.channel("vae") if comm is not None else None)
    elif not args.no_decode:                       # ftlk (C1): the reference's orthogonal codec
        from paper_2512_23379_b200.codec import Codec
        vae = Codec(np.linalg.qr(np.random.default_rng(0).standard_normal((cfg.latent_dim, cfg.latent_dim)))[0])

    from paper_2512_23379_b200.streaming import DeviceStreamer

    class _Runner:   # DeviceStreamer over the synthetic-weight denoiser
        pass
    runner = _Runner()
    runner.cfg, runner.device = cfg, dev
    runner.denoiser = lambda lc, lm, hw: d
    ds = DeviceStreamer(runner, scfg, vae, ref_host, lat_hw, use_graph=not args.no_graph)
    # inputs resident in HBM before the timed region: per-chunk noise and staged cond inputs
    z_all, cond_all = [], []
    for c in range(nsteps):
        z_all.append(torch.as_tensor(chunk_noise(0, c, (S,) + fshape), dtype=torch.float32, device=dev))
        d.stage_cond(windows[c], ref_host, 0)
        cond_all.append(d._cond_stage[0].to(dev))

    marks = []   # per-chunk (start, denoised, decode start, decoded) events: component split for latency.py
    overlap = vae is not None and args.overlap
    dstream = torch.cuda.Stream(device=dev) if overlap else stream
    slots = [torch.empty_like(ds.x0_static) for _ in range(2)] if overlap else None
    freed = [None, None]

    def chunk(c, mark=False):
        """One chunk. With overlap (the engine's schedule: streaming.StreamSession decodes on its
        own stream), chunk c's decode runs on a second stream while chunk c+1 denoises."""
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if mark else None
        if mark:
            ev[0].record(stream)
        x0 = ds.run_resident(z_all[c], cond_all[c])
        if overlap:
            k = c & 1
            if freed[k] is not None:
                stream.wait_event(freed[k])        # decode of chunk c-2 done with this slot
            slots[k].copy_(x0)
            x0 = slots[k]
        if mark:
            ev[1].record(stream)
        if overlap:
            dstream.wait_stream(stream)
        if mark:
            ev[2].record(dstream)
        if vae is not None:   # N > 1: the decoded slabs are gathered into rank 0's frames
            with torch.cuda.stream(dstream):
                vae.decode_device_tensor(x0, dstream, gather=True)
            if overlap:
                freed[c & 1] = torch.cuda.Event()
                freed[c & 1].record(dstream)
        if mark:
            ev[3].record(dstream)
            marks.append(ev)

    def drain():
        if overlap:
            stream.wait_stream(dstream)

    # ---------------- warm-up (also fills the per-ladder AdaLN cache)
    for c in range(args.warmup):
        chunk(c)
    drain()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = _capi.LAUNCHES[0]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for c in range(args.warmup, nsteps):
        chunk(c, mark=True)
    drain()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = _capi.LAUNCHES[0] - launches0 + (ds.graph_launches * args.steps if ds.graph is not None else 0)
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    clk = clocks.stop()
    fps = frames_per_chunk * 1000.0 / ms   # one stream sharded over all ranks (strong scaling)
    comp = {"denoise": float(np.mean([a.elapsed_time(b) for a, b, _, _ in marks])),
            "decode": float(np.mean([c.elapsed_time(d) for _, _, c, d in marks])),
            "latency": float(np.mean([a.elapsed_time(d) for a, _, _, d in marks])),
            "decode_overlaps_denoise": overlap,
            "steps_per_chunk": scfg.sampler.steps, "frames_per_chunk": frames_per_chunk}

    # ---------------- e2e through the public engine API: a StreamSession (start_stream) on the same
    # device weights, driven with host samples (push_signal) and drained frame by frame (next_frames):
    # host PCG64 noise, pinned H2D of noise + window, the decode on the session's own stream, D2H of
    # the RGB8 frames, the engine's three threads. Wall time on rank 0 from the first push of the
    # timed chunks to the last frame, max over ranks (followers run in lockstep through the gather).
    e2e = None
    if not args.no_e2e:
        from paper_2512_23379_b200.streaming import start_stream
        sess = start_stream(w, cfg, vae, None, scfg, reference_latent=ref_host, latent_hw=lat_hw, comm=comm)
        hsync = comm.host_channel("bench") if comm is not None else None
        rs = np.random.default_rng(11)
        samples = (rs.standard_normal((nsteps * S, A, adim)) if cfg.mode == "wan"
                   else rs.uniform(-1, 1, nsteps * S))
        d2h = [0]

        def run_chunks(c0, c1):
            if rank == 0:
                sess.push_signal((i, samples[i]) for i in range(c0 * S, c1 * S))
                need, n = (c1 - c0) * frames_per_chunk, 0
                while n < need:
                    fr, _ = sess.next_frames(wait=True, timeout=1.0)
                    n += len(fr)
                    if fr:
                        d2h[0] = int(np.asarray(fr[0].state).nbytes) * frames_per_chunk
            if hsync is not None:
                hsync.host_broadcast(None)      # followers wait here (gloo) while their session threads run
        run_chunks(0, args.warmup)
        t0 = time.perf_counter()
        run_chunks(args.warmup, nsteps)
        ems = max_over_ranks((time.perf_counter() - t0) * 1000.0 / args.steps)
        sess.close()
        h2d = ds.noise_host[0].numel() * 4 + d.buf["cond_in"].numel() * 2
        e2e = {"value": frames_per_chunk * 1000.0 / ems, "unit": "FPS", "ms_per_step": ems,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h[0],
               "api": "streaming.start_stream -> StreamSession.push_signal / next_frames (unpaced, host wall time)"}

    # ---------------- instrumented chunk: per-kernel durations for the roofline
    ops.PROFILER = []
    ops.PROFILE_DETAIL = True               # per-shape kinds ("gemm:qkv_rope:MxNxK", "conv:...")
    ds.z.copy_(z_all[nsteps - 1])
    ds.d.buf["cond_in"].copy_(cond_all[nsteps - 1])
    ds._device_chunk()                      # eager: every launch bracketed by events
    if vae is not None:
        vae.decode_device_tensor(ds.x0_static, stream, gather=True)
    torch.cuda.synchronize()
    prof = ops.PROFILER
    ops.PROFILER = None
    ops.PROFILE_DETAIL = None
    det, agg = {}, {}
    for kind, a, b, fl, nb in prof:
        t = a.elapsed_time(b)
        for key, table in ((kind, det), (kind.split(":")[0], agg)):
            g = table.setdefault(key, [0.0, 0.0, 0.0, 0])
            g[0] += t
            g[1] += fl
            g[2] += nb
            g[3] += 1
    if args.detail:
        for k, v in sorted(det.items(), key=lambda kv: -kv[1][0]):
            sys.stderr.write("%-50s %9.3f ms %5d launches %8.1f TFLOP/s\n" % (
                k, v[0], v[3], v[1] / (v[0] * 1e-3) / 1e12 if v[1] else 0.0))
    pk, pk_src = peaks()
    peak = pk["bf16_tflops_sustained"]
    # dominant kernel: the tcgen05 GEMM at its largest launch (QKV projection + RoPE epilogue)
    qkv = [(k, v) for k, v in det.items() if k.startswith("gemm:qkv_rope")]
    qk, qv = max(qkv, key=lambda kv: kv[1][1]) if qkv else max(
        ((k, v) for k, v in det.items() if k.startswith("gemm")), key=lambda kv: kv[1][1])
    q_ms = qv[0] / qv[3]
    q_flops = qv[1] / qv[3]
    ach = q_flops / (q_ms * 1e-3) / 1e12
    traffic, traffic_src = None, None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))["kernels"]["gemm"]
        if qk.split(":")[-1] in tr["shape"].replace(" ", ""):
            traffic, traffic_src = tr["dram_bytes"], "profiles/ncu_traffic.json (%s, ncu --set full)" % tr["shape"]
    except Exception:  # noqa: BLE001
        pass
    gem = agg.get("gemm", [1e-9, 0, 0, 1])
    conv = agg.get("conv", [1e-9, 0, 0, 1])
    breakdown = {k: {"ms": v[0], "launches": v[3], "tflops": (v[1] / (v[0] * 1e-3) / 1e12) if v[1] else None,
                     "gbs": (v[2] / (v[0] * 1e-3) / 1e9)} for k, v in agg.items()}
    dit_flops = sum(v[1] for k, v in agg.items() if k != "conv")
    roofline = {"bound": "tensor", "kernel": "ftb gemm_tc_pair_kernel, %s" % qk,
                "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                "peak_source": pk_src + " bf16_tflops_sustained (kernel timed inside the chunk)",
                "traffic": traffic, "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": qv[2] / qv[3],
                "flops_per_launch": q_flops, "avg_launch_ms": q_ms, "launches_per_chunk": qv[3],
                "all_gemms_tflops": gem[1] / (gem[0] * 1e-3) / 1e12,
                "dit_chunk_flops": dit_flops, "dit_tflops_achieved": dit_flops / (comp["denoise"] * 1e-3) / 1e12,
                "dit_frac": dit_flops / (comp["denoise"] * 1e-3) / 1e12 / peak, "per_kind": breakdown,
                "vae_conv_tflops": conv[1] / (conv[0] * 1e-3) / 1e12 if conv[1] else None}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and cfg.mode == "wan":
        from oracle.cpu_baseline import extrapolated_chunk_seconds
        T = d.T
        chunk_s, det = extrapolated_chunk_seconds(cfg.model_dim, cfg.heads, cfg.ff_dim, cfg.layers, 4, d.L, T)
        cpu = {"value": frames_per_chunk / chunk_s, "unit": "FPS", "cores": os.cpu_count(), "kind": "port",
               "sample": "one %s-width wan layer fwd (fp64 NumPy oracle) on one latent frame (%d of %d tokens), "
                         "self-attention core on %d of %d heads, extrapolated to %d layers x 4 steps (DiT only)" % (
                             args.model, det["L_sample"], d.L, det["attn_heads_timed"], cfg.heads, cfg.layers),
               "chunk_seconds": chunk_s}
    elif rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            t = reference_tiny_chunks(200, "cython")
            chunk_s = float(np.median(t))
            cpu = {"value": frames_per_chunk / chunk_s, "unit": "FPS", "cores": 1, "kind": "reference",
                   "sample": "ftlk rollout_stream + Codec.decode (baseline/_ref, cython backend), median of 200 "
                             "chunks", "chunk_seconds": chunk_s}
        except ImportError as e:
            cpu = {"value": None, "unit": "FPS", "cores": 0, "kind": "reference", "sample": "unavailable: %s" % e}

    if rank == 0:
        line = {"metric": "streaming FPS (%s-shape DiT, 4-step chunk, %d frames/chunk)" % (
                    {"14b": "14B", "1.3b": "1.3B", "tiny": "tiny ftlk"}[args.model], frames_per_chunk), "value": fps,
                "unit": "FPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "chunk_latency_ms": comp["latency"], "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, N(0,1) audio)",
                "config": {"workload": workload_name(args), "model": args.model, "layers": cfg.layers,
                           "model_dim": cfg.model_dim, "heads": cfg.heads, "global_batch": 1,
                           "seq_len": d.L, "latent_grid": list(lat_hw), "frames_per_chunk": frames_per_chunk,
                           "parallelism": "ulysses_sp%d" % world if world > 1 else "single",
                           "comm": comm_note, "cuda_graph": ds.graph is not None,
                           "decode": "causal VAE decoder, 7 latents -> 28 RGB8 frames %dx%d" % (Hpx, Wpx)
                           if vae is not None else "none",
                           "l2": "working set > L2 (weights %.1f GB)" % (w.nbytes() / 1e9)},
                "components_ms": comp,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk}
        ovr = {k: os.environ[k] for k in ("FTB_GEMM_VARIANT", "FTB_GEMM_GROUP", "FTB_CONV_VARIANT", "FTB_ATTN_NO_SPLIT")
               if os.environ.get(k)}
        if ovr:   # A/B run with non-default kernel variants: say so in the line
            line["config"]["kernel_overrides"] = ovr
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
