"""Multi-process host logic of the Ulysses path on CPU (gloo, world_size 2):
shard plan arithmetic and the collective layouts the device path relies on."""

import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2512_23379_b200.dist import ShardPlan


def test_shard_plan_arithmetic():
    for L, g in [(10530, 1), (10530, 2), (10530, 4), (10530, 8), (162, 4), (9, 2)]:
        plans = [ShardPlan(L, g, r) for r in range(g)]
        assert all(p.Ls * g == p.L_pad >= L for p in plans)
        assert plans[0].L_pad - L < g
        assert sum(p.valid for p in plans) == L
        assert [p.start for p in plans] == [r * plans[0].Ls for r in range(g)]
    assert ShardPlan(10530, 8, 0).Ls == 1317
    assert ShardPlan(10530, 8, 0).heads_per_rank(40) == 5
    with pytest.raises(Exception):
        ShardPlan(10530, 8, 0).heads_per_rank(12)


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2512_23379_b200.dist import TorchComm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        Ls, hw, L = 3, 4, 5          # L_pad = 6
        # QKV send layout [dest][Ls][3][hw]; value encodes (src rank, dest, local token, which, d)
        send = torch.zeros(world, Ls, 3, hw)
        for dst in range(world):
            for t in range(Ls):
                for w in range(3):
                    send[dst, t, w] = torch.arange(hw, dtype=torch.float32) + 1000 * rank + 100 * dst + 10 * t + w * 0.1
        recv = torch.empty(world * Ls, 3, hw)
        comm.all_to_all(recv, send)
        # full sequence for my head group: token rows in global order
        for src in range(world):
            for t in range(Ls):
                exp = torch.arange(hw, dtype=torch.float32) + 1000 * src + 100 * rank + 10 * t
                assert torch.allclose(recv[src * Ls + t, 0], exp)
        out = torch.empty(world * Ls, 2)
        comm.all_gather(out, torch.full((Ls, 2), float(rank)))
        assert torch.equal(out[:Ls], torch.zeros(Ls, 2)) and torch.equal(out[Ls:], torch.ones(Ls, 2))
        q.put((rank, "ok", L))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e), 0))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_collective_layouts():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 300
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res


def _halo_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2512_23379_b200.dist import TorchComm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        first = torch.full((4, 6), 10.0 * rank + 1)
        last = torch.full((4, 6), 10.0 * rank + 2)
        top, bot = torch.empty(4, 6), torch.empty(4, 6)
        comm.neighbor_exchange(first, last, top, bot)
        exp_top = 0.0 if rank == 0 else 10.0 * (rank - 1) + 2
        exp_bot = 0.0 if rank == world - 1 else 10.0 * (rank + 1) + 1
        assert torch.all(top == exp_top) and torch.all(bot == exp_bot), (rank, top[0, 0], bot[0, 0])
        q.put((rank, "ok", 0))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e), 0))
    finally:
        dist.destroy_process_group()


def test_gloo_halo_exchange_world3():
    """Spatially split VAE: edge-row swap with neighbours, zeros at the global edges."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29900 + os.getpid() % 90
    ps = [ctx.Process(target=_halo_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res


def _engine_io_worker(rank, world, port, q):
    """Host plumbing of the multi-rank engine: the ingest channel's chunk broadcast (rank 0 ->
    followers, end-of-stream sentinel), a decode channel independent of the DiT group, and the
    frame gather of row slabs into rank 0 (uneven slabs)."""
    import torch.distributed as dist

    from paper_2512_23379_b200.dist import TorchComm, slab_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        host = comm.host_channel("ingest")
        vae = comm.channel("vae")
        assert (host.world, host.rank, vae.world, vae.rank) == (world, rank, world, rank)
        windows = [np.full((3, 2), 0.5 * c) for c in range(4)]
        seen = []
        for c in range(5):
            item = host.host_broadcast((c, windows[c]) if c < 4 else None) if rank == 0 else host.host_broadcast(None)
            if item is None:
                break
            seen.append(item)
        assert [c for c, _ in seen] == [0, 1, 2, 3]
        assert all(np.array_equal(w, windows[c]) for c, w in seen)
        sizes = slab_rows(7, world)
        r0 = sum(sizes[:rank])
        slab = torch.arange(r0, r0 + sizes[rank], dtype=torch.float32).view(1, -1, 1, 1).expand(2, -1, 3, 2).clone()
        full = torch.full((2, 7, 3, 2), -1.0)
        vae.gather_rows("frames", full, slab, sizes)
        if rank == 0:
            want = torch.arange(7, dtype=torch.float32).view(1, 7, 1, 1).expand(2, 7, 3, 2)
            assert torch.equal(full, want)
        # every rank gets every slab (the decoder mid attention's keys / values)
        full2 = torch.full((2, 7, 3, 2), -1.0)
        vae.all_gather_rows("kv", full2, slab, sizes)
        assert torch.equal(full2, torch.arange(7, dtype=torch.float32).view(1, 7, 1, 1).expand(2, 7, 3, 2))
        q.put((rank, "ok", 0))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e), 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_engine_host_plumbing(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30100 + world * 50 + os.getpid() % 40
    ps = [ctx.Process(target=_engine_io_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res


def test_slab_rows_partition():
    from paper_2512_23379_b200.dist import slab_rows
    assert slab_rows(52, 8) == [7, 7, 7, 7, 6, 6, 6, 6]
    assert slab_rows(90, 8) == [12, 12, 11, 11, 11, 11, 11, 11]
    assert sum(slab_rows(9, 8)) == 9
    with pytest.raises(Exception):
        slab_rows(5, 8)
