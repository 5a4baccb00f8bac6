"""Multi-process peer transport on one B200: two processes (gloo process group for
the handle exchange and a host barrier, so no kernel ever waits on another
process's kernel) run the Ulysses step with the QKV / FMHA / out-projection
epilogues storing through cudaIpc-imported peer pointers; both ranks must
reproduce the single-process step."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _setup():
    from paper_2512_23379_b200.config import NetConfig
    from paper_2512_23379_b200.net import ParamStore
    cfg = NetConfig(256, 2, 4, 512, 16, mode="wan", patch=(1, 2, 2), audio_dim=16, audio_tokens=2)
    store = ParamStore.init(cfg, 5)
    r = np.random.default_rng(5)
    x = dict(motion=r.standard_normal((1, 16, 12, 18)), z=r.standard_normal((2, 16, 12, 18)),
             ref=r.standard_normal((16, 12, 18)), audio=r.standard_normal((3, 2, 16)))
    return cfg, store, x


def _step(comm):
    from paper_2512_23379_b200.model import DeviceDenoiser, DeviceWeights
    cfg, store, x = _setup()
    dev = torch.device("cuda", 0)
    w = DeviceWeights.from_host(cfg, store.params, dev)
    s = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(s):
        d = DeviceDenoiser(w, 3, 1, (12, 18), stream=s, comm=comm)
        d.prepare_cond(x["audio"], x["ref"])
        fv = d.frame_vectors(np.array([0.0, 0.75, 0.75]))
        args = [torch.as_tensor(x[k], dtype=torch.float32, device=dev) for k in ("motion", "z", "ref")]
        for _ in range(2):   # two steps: receive buffers reused across steps and layers
            x0t = d.step(*args, fv)
        out = d.tokens_to_frames(x0t).double().cpu().numpy()
    s.synchronize()
    return out


def _worker(rank, world, port, outdir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_23379_b200.dist import IpcPeerComm
    comm = IpcPeerComm(torch.device("cuda", 0), barrier_mode="host")
    out = _step(comm)
    np.save(os.path.join(outdir, "r%d.npy" % rank), out)
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


def _reference(outdir):
    np.save(os.path.join(outdir, "ref.npy"), _step(None))


def test_ipc_peer_transport_two_processes(cuda, tmp_path):
    # every CUDA step runs in a spawned child (the single-process reference too): the pytest
    # process itself stays out of this test's multi-process CUDA work
    ctx = mp.get_context("spawn")
    ref = ctx.Process(target=_reference, args=(str(tmp_path),))
    ref.start()
    ref.join(timeout=600)
    assert ref.exitcode == 0
    want = np.load(tmp_path / "ref.npy")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    for r in range(2):
        got = np.load(tmp_path / ("r%d.npy" % r))
        rel = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert rel < 5e-3, (r, rel)
