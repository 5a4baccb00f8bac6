"""The streaming engine across ranks (north star "8xB200"): g ranks emulated on one
B200 (one thread per rank, host-barrier transports: no kernel ever waits on another). Rank 0
pushes the driving signal, the followers receive every chunk's window over the host channel,
the DiT runs Ulysses over the ranks, the causal VAE decodes one row slab per rank on its own
channel and gathers the frames into rank 0, which alone emits them. The emitted frames must
match the single-GPU session's (same indices, RGB8 within rounding) on both transports."""

import threading
import time

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

VAE = dict(z_dim=16, base_dim=32, dim_mult=(1, 2, 4, 4), num_res_blocks=2, temporal_upsample=(True, True, False))


def _setup():
    from paper_2512_23379_b200.config import NetConfig
    from paper_2512_23379_b200.net import ParamStore
    from paper_2512_23379_b200.vae import VAEConfig, init_vae_params
    cfg = NetConfig(512, 2, 8, 1024, 16, mode="wan", patch=(1, 2, 2), audio_dim=16, audio_tokens=2)   # hd 64
    store = ParamStore.init(cfg, 5)
    vcfg = VAEConfig(**VAE)
    P = init_vae_params(vcfg, 4)
    r = np.random.default_rng(9)
    H, W = 12, 16
    ref = r.standard_normal((16, H, W))
    signal = r.standard_normal((14, 2, 16))
    return cfg, store, vcfg, P, ref, signal, (H, W)


def _run(world, transport, dev):
    """One session per rank; returns (rank 0's emitted frames, per-rank stats)."""
    from paper_2512_23379_b200.config import StreamConfig
    from paper_2512_23379_b200.dist import ThreadComm, ThreadPeerComm
    from paper_2512_23379_b200.streaming import start_stream
    from paper_2512_23379_b200.vae import DeviceVAEDecoder
    cfg, store, vcfg, P, ref, signal, hw = _setup()
    comms = (ThreadPeerComm if transport == "peer" else ThreadComm).make(world) if world > 1 else [None]
    got, stats, errs = [], [None] * world, []
    done = threading.Event()
    n_frames = 2 * 7 * 4

    def rank_main(r):
        try:
            torch.cuda.set_device(dev)
            comm = comms[r]
            dec = DeviceVAEDecoder(vcfg, dev, params=P, rgb8=True,
                                   comm=comm.channel("vae") if comm is not None else None)
            sess = start_stream(store, cfg, dec, None, StreamConfig(seed=3), reference_latent=ref,
                                latent_hw=hw, comm=comm)
            if r == 0:
                sess.push_signal((i, signal[i]) for i in range(len(signal)))
                deadline = time.time() + 240
                while len(got) < n_frames and time.time() < deadline:
                    fr, _ = sess.next_frames(wait=True, timeout=0.2)
                    got.extend(fr)
                done.set()
            else:
                with pytest.raises(Exception):
                    sess.push_signal([(0, signal[0])])     # followers take rank 0's schedule
                done.wait(300)
            stats[r] = sess.stats()
            sess.close()
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            done.set()
            raise
    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=400)
    assert not errs, errs
    return got, stats


@pytest.mark.parametrize("world,transport", [(2, "coll"), (2, "peer"), (8, "peer")])
def test_stream_session_ranks_match_one(cuda, world, transport):
    """g = 8: 8 heads (one per rank), 12 latent rows split 2,2,2,2,1,1,1,1."""
    one, _ = _run(1, None, cuda)
    two, st = _run(world, transport, cuda)
    assert [f.index for f in two] == [f.index for f in one] == list(range(56))
    assert [f.chunk for f in two] == [f.chunk for f in one]
    a = np.stack([f.state for f in one]).astype(int)
    b = np.stack([f.state for f in two]).astype(int)
    assert a.shape == b.shape == (56, 96, 128, 3)
    assert np.mean(np.abs(a - b) <= 2) > 0.99
    assert st[0].frames_emitted == 56 and all(x.frames_emitted == 0 for x in st[1:])   # only rank 0 emits


def test_generate_two_ranks_matches_one(cuda):
    """Synchronous generate() with a communicator: every rank calls it with the same inputs;
    targets are replicated, the gathered frames come back on rank 0."""
    from paper_2512_23379_b200.config import StreamConfig
    from paper_2512_23379_b200.dist import ThreadPeerComm
    from paper_2512_23379_b200.streaming import generate
    from paper_2512_23379_b200.vae import DeviceVAEDecoder
    cfg, store, vcfg, P, ref, signal, hw = _setup()
    dec = DeviceVAEDecoder(vcfg, cuda, params=P, rgb8=False)
    t1, _, f1 = generate(store, cfg, dec, ref, signal, 14, cfg=StreamConfig(seed=3), latent_hw=hw)
    comms = ThreadPeerComm.make(2)
    out, errs = [None, None], []

    def rank_main(r):
        try:
            torch.cuda.set_device(cuda)
            d = DeviceVAEDecoder(vcfg, cuda, params=P, rgb8=False, comm=comms[r].channel("vae"))
            s = torch.cuda.Stream(device=cuda)
            with torch.cuda.stream(s):
                out[r] = generate(store, cfg, d, ref, signal, 14, cfg=StreamConfig(seed=3), latent_hw=hw,
                                  comm=comms[r])
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            raise
    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errs, errs
    (ta, _, fa), (tb, _, fb) = out
    assert np.array_equal(ta, tb)                     # replicated sampler state
    rel = float(np.linalg.norm(ta - t1) / np.linalg.norm(t1))
    assert rel < 5e-3
    assert fb is None and fa is not None and fa.shape == f1.shape
    frel = float(np.linalg.norm(fa[..., :3] - f1[..., :3]) / np.linalg.norm(f1[..., :3]))
    assert frel < 5e-3
