"""Ulysses sequence parallelism, g ranks emulated on one B200 (one thread per
rank, ThreadComm exchanges, no kernel ever waits on another): the sharded step
must reproduce the single-rank step and the oracle."""

import threading

import numpy as np
import pytest
import torch

from oracle import wan_oracle as WO

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _setup(heads=4, hd=64, Lc=3, Lm=1, H=12, W=18, layers=2, seed=5):
    from paper_2512_23379_b200.config import NetConfig
    from paper_2512_23379_b200.net import ParamStore
    m = heads * hd
    cfg = NetConfig(m, layers, heads, 2 * m, 16, mode="wan", patch=(1, 2, 2), audio_dim=16, audio_tokens=2)
    store = ParamStore.init(cfg, seed)
    r = np.random.default_rng(seed)
    x = dict(motion=r.standard_normal((Lm, 16, H, W)), z=r.standard_normal((Lc - Lm, 16, H, W)),
             ref=r.standard_normal((16, H, W)), audio=r.standard_normal((Lc, 2, 16)))
    return cfg, store, x, (Lc, Lm, H, W)


def _run(cfg, store, x, geo, world, dev, transport="coll"):
    from paper_2512_23379_b200.dist import ThreadComm, ThreadPeerComm
    from paper_2512_23379_b200.model import DeviceDenoiser, DeviceWeights
    Lc, Lm, H, W = geo
    w = DeviceWeights.from_host(cfg, store.params, dev)
    make = ThreadPeerComm.make if transport == "peer" else ThreadComm.make
    comms = make(world) if world > 1 else [None]
    out, errs = [None] * world, []
    frame_t = np.where(np.arange(Lc) < Lm, 0.0, 0.75)

    def worker(r):
        try:
            torch.cuda.set_device(dev)
            s = torch.cuda.Stream(device=dev)
            with torch.cuda.stream(s):
                d = DeviceDenoiser(w, Lc, Lm, (H, W), stream=s, comm=comms[r])
                md = torch.as_tensor(x["motion"], dtype=torch.float32, device=dev)
                zd = torch.as_tensor(x["z"], dtype=torch.float32, device=dev)
                rd = torch.as_tensor(x["ref"], dtype=torch.float32, device=dev)
                d.prepare_cond(x["audio"], x["ref"])
                fv = d.frame_vectors(frame_t)
                x0t = d.step(md, zd, rd, fv)
                out[r] = d.tokens_to_frames(x0t).double().cpu().numpy()
                s.synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            raise
    ts = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errs, errs
    return out, frame_t


def _setup_for(world):
    # 8 ranks need 8 heads; L = 3 * 6 * 9 = 162 tokens is not a multiple of 4 or 8 (padded shards)
    return _setup(heads=8, hd=64) if world == 8 else _setup()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_ulysses_matches_single_rank(cuda, world):
    cfg, store, x, geo = _setup_for(world)
    one, frame_t = _run(cfg, store, x, geo, 1, cuda)
    many, _ = _run(cfg, store, x, geo, world, cuda)
    for r in range(world):
        assert rel(many[r], one[0]) < 5e-3, r   # same kernels; short shards may pick the CUDA-core cross-attn
    ref = WO.denoise(store.bf16_rounded().params, dict(model_dim=cfg.model_dim, layers=cfg.layers, heads=cfg.heads,
                                                       latent_dim=16, patch=(1, 2, 2), audio_tokens=2, audio_dim=16),
                     x["motion"], x["z"], x["ref"], x["audio"], frame_t)
    assert rel(many[0], ref) < 1e-2


@pytest.mark.parametrize("world", [2, 4, 8])
def test_ulysses_peer_epilogues_match_collectives(cuda, world):
    """Fused transport (QKV / FMHA / out-projection epilogues storing into the peers'
    receive buffers, barrier after each producer) == the NCCL-style collective
    transport, bit for bit: same kernels, same operands, only the store targets move."""
    cfg, store, x, geo = _setup_for(world)
    coll, _ = _run(cfg, store, x, geo, world, cuda, "coll")
    peer, _ = _run(cfg, store, x, geo, world, cuda, "peer")
    for r in range(world):
        assert np.array_equal(peer[r], coll[r]), r
    assert all(np.array_equal(peer[r], peer[0]) for r in range(world))   # replicated x0


@pytest.mark.parametrize("world", [4, 8])
def test_ulysses_peer_padding_path(cuda, world):
    cfg, store, x, geo = _setup_for(world)
    assert (geo[0] * (geo[2] // 2) * (geo[3] // 2)) % world != 0
    one, _ = _run(cfg, store, x, geo, 1, cuda)
    many, _ = _run(cfg, store, x, geo, world, cuda, "peer")
    for r in range(world):
        assert rel(many[r], one[0]) < 5e-3, r


def test_peer_barrier_kernel_single_rank(cuda):
    """Device barrier mechanics at world 1 (signals and waits on itself): the epoch
    counter advances once per call, also when replayed from a CUDA graph."""
    from paper_2512_23379_b200 import ops
    flags = torch.zeros(1, dtype=torch.int32, device=cuda)
    epoch = torch.zeros(1, dtype=torch.int32, device=cuda)
    for _ in range(3):
        ops.peer_barrier([flags.data_ptr()], epoch, 0, 1, 5.0)
    torch.cuda.synchronize()
    assert int(epoch.item()) == 3 and int(flags.item()) == 3
    s = torch.cuda.Stream(device=cuda)
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ops.peer_barrier([flags.data_ptr()], epoch, 0, 1, 5.0)
        ops.peer_barrier([flags.data_ptr()], epoch, 0, 1, 5.0)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    assert int(epoch.item()) == 7 and int(flags.item()) == 7


def test_ulysses_padding_path(cuda):
    """L = 3*6*9 = 162 tokens: not divisible by 4 -> padded shards, masked keys."""
    cfg, store, x, geo = _setup(Lc=3, Lm=1, H=12, W=18)
    assert (geo[0] * (geo[2] // 2) * (geo[3] // 2)) % 4 != 0
    one, _ = _run(cfg, store, x, geo, 1, cuda)
    many, _ = _run(cfg, store, x, geo, 4, cuda)
    assert rel(many[3], one[0]) < 5e-3


SMALL_VAE = dict(z_dim=16, base_dim=32, dim_mult=(1, 2, 4, 4), num_res_blocks=2, temporal_upsample=(True, True, False))


@pytest.mark.parametrize("transport", ["coll", "peer"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_split_vae_matches_unsplit(cuda, world, transport):
    """Spatially split causal VAE decode (row slabs + per-conv halo exchange, two
    chunks so the causal caches of slabs and halos are exercised) == unsplit decode;
    halos through collectives or stored into the neighbours' buffers (peer transport)."""
    from paper_2512_23379_b200.dist import ThreadComm, ThreadPeerComm
    from paper_2512_23379_b200.vae import DeviceVAEDecoder, VAEConfig, init_vae_params
    cfg = VAEConfig(**SMALL_VAE)
    P = init_vae_params(cfg, 4)
    r = np.random.default_rng(1)
    zs = [r.standard_normal((3, 16, 9 if world == 8 else 6, 8)) for _ in range(2)]   # g=8: 2,1,..,1 rows
    ref_dec = DeviceVAEDecoder(cfg, cuda, params=P, rgb8=False)
    want = [ref_dec.decode_device(torch.as_tensor(z, dtype=torch.float32, device=cuda), torch.cuda.current_stream())
            for z in zs]
    comms = (ThreadPeerComm if transport == "peer" else ThreadComm).make(world)
    got, errs = [[None] * world for _ in zs], []

    def worker(rk):
        try:
            torch.cuda.set_device(cuda)
            s = torch.cuda.Stream(device=cuda)
            dec = DeviceVAEDecoder(cfg, cuda, params=P, rgb8=False, comm=comms[rk])
            for i, z in enumerate(zs):
                with torch.cuda.stream(s):
                    zd = torch.as_tensor(z, dtype=torch.float32, device=cuda)
                    full = dec.decode_device_tensor(zd, s, gather=True)  # frames gathered into rank 0
                    full = None if full is None else full.clone()
                    slab = dec.last_slab.clone()                         # this rank's row slab
                s.synchronize()
                got[i][rk] = (dec.row0, slab.cpu().numpy(), None if full is None else full.cpu().numpy())
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            raise
    ts = [threading.Thread(target=worker, args=(k,)) for k in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errs, errs
    for i in range(2):
        slabs = sorted(got[i], key=lambda x: x[0])
        cat = np.concatenate([sl for _, sl, _ in slabs], axis=1)
        assert cat[..., :3].shape == want[i][..., :3].shape
        assert rel(cat[..., :3], want[i][..., :3]) < 2e-3, i
        gathered = [fg for _, _, fg in got[i] if fg is not None]
        assert len(gathered) == 1 and np.array_equal(gathered[0], cat)   # rank 0 alone gets all slabs


@pytest.mark.parametrize("transport", ["coll", "peer"])
def test_split_vae_rgb8_head_equals_unsplit(cuda, transport):
    """RGB8 decode (head as 1x1 GEMM + 27-tap gather, halo rows through their own GEMM blocks),
    split over 3 ranks and gathered into rank 0 == the unsplit RGB8 decode, byte for byte."""
    from paper_2512_23379_b200.dist import ThreadComm, ThreadPeerComm
    from paper_2512_23379_b200.vae import DeviceVAEDecoder, VAEConfig, init_vae_params
    cfg = VAEConfig(**SMALL_VAE)
    P = init_vae_params(cfg, 6)
    r = np.random.default_rng(2)
    zs = [r.standard_normal((3, 16, 7, 9)) for _ in range(2)]
    ref = DeviceVAEDecoder(cfg, cuda, params=P, rgb8=True)
    want = [ref.decode_device(torch.as_tensor(z, dtype=torch.float32, device=cuda), torch.cuda.current_stream())
            for z in zs]
    world = 3
    comms = (ThreadPeerComm if transport == "peer" else ThreadComm).make(world)
    got, errs = [None, None], []

    def worker(rk):
        try:
            torch.cuda.set_device(cuda)
            s = torch.cuda.Stream(device=cuda)
            dec = DeviceVAEDecoder(cfg, cuda, params=P, rgb8=True, comm=comms[rk])
            for i, z in enumerate(zs):
                with torch.cuda.stream(s):
                    zd = torch.as_tensor(z, dtype=torch.float32, device=cuda)
                out = dec.decode_device(zd, s)
                if rk == 0:
                    got[i] = out
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            raise
    ts = [threading.Thread(target=worker, args=(k,)) for k in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errs, errs
    for i in range(2):
        assert got[i].dtype == np.uint8 and np.array_equal(got[i], want[i]), i


@pytest.mark.parametrize("world", [2, 4, 8])
def test_peer_barrier_protocol_concurrent_ranks(cuda, world):
    """The device barrier's protocol (release-store of the epoch into every rank's flag word,
    acquire-spin on its own) with `world` truly concurrent ranks: one co-resident block per rank
    in a cooperative launch (never separate launches that wait on one another on one GPU).
    Every round's payload of every rank is visible after the barrier; the epochs advance once
    per barrier."""
    from paper_2512_23379_b200 import _capi as A
    rounds = 2000
    flags = torch.zeros(world * world, dtype=torch.int32, device=cuda)
    epochs = torch.zeros(world, dtype=torch.int32, device=cuda)
    data = torch.zeros(rounds * world, dtype=torch.int32, device=cuda)
    errors = torch.zeros(1, dtype=torch.int32, device=cuda)
    A.call("ftb_peer_barrier_selftest", world, rounds, A.ptr(flags), A.ptr(epochs), A.ptr(data), A.ptr(errors),
           10.0, A.stream_ptr())
    torch.cuda.synchronize()
    assert int(errors.item()) == 0
    assert torch.all(epochs == 2 * rounds)
    assert torch.all(flags == 2 * rounds)
