"""Ulysses sequence parallelism for the DiT step.

One process per GPU. The chunk's L tokens (frame-major) are padded to
L_pad = ceil(L / g) * g and split into g equal contiguous shards; rank r owns
tokens [r*Ls, (r+1)*Ls). Weights are replicated. Per layer:

  QKV GEMM on the local shard; its epilogue writes the send layout
  [dest][Ls][3][H/g][hd] (dest = head group)            -- no pack kernel
  all-to-all #1  -> [L_pad][3][H/g][hd]  (full sequence, own head group)
  flash attention over H/g heads, keys >= L masked
  all-to-all #2  -> [src head group][Ls][H/g*hd]
  O GEMM reads the g head-group slices directly (3D TMA map, `a_chunks=g`)

Cross-attention K/V (conditioning tokens) and the AdaLN tables are replicated,
so they need no exchange; after the out-projection the x0 tokens are
all-gathered so every rank applies the same DDIM update (replicated sampler
state). Communication is NCCL over NVLink through torch.distributed; a
thread-based emulation (`ThreadComm`) runs g ranks on one device for tests.
"""

import threading

import torch

from .errors import ConfigError


class ShardPlan:
    """Token partition of one chunk for g ranks."""

    def __init__(self, L, world, rank):
        if world < 1 or not (0 <= rank < world):
            raise ConfigError("bad world/rank")
        self.L, self.world, self.rank = int(L), int(world), int(rank)
        self.Ls = -(-self.L // self.world)
        self.L_pad = self.Ls * self.world
        self.start = self.rank * self.Ls
        self.valid = max(0, min(self.Ls, self.L - self.start))  # real tokens in this shard

    def heads_per_rank(self, heads):
        if heads % self.world:
            raise ConfigError("heads (%d) must divide by the Ulysses degree (%d)" % (heads, self.world))
        return heads // self.world

    def __repr__(self):
        return "ShardPlan(L=%d, world=%d, rank=%d, Ls=%d, pad=%d)" % (self.L, self.world, self.rank, self.Ls,
                                                                       self.L_pad - self.L)


class LocalComm:
    world, rank = 1, 0

    def neighbor_exchange(self, send_first, send_last, recv_top, recv_bot, stream=None):
        recv_top.zero_()
        recv_bot.zero_()

    def all_to_all(self, out, inp, stream=None):
        out.copy_(inp)

    def all_gather(self, out, inp, stream=None):
        out.copy_(inp)


class TorchComm:
    """torch.distributed (NCCL on GPUs, gloo on CPU) equal-split collectives."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_to_all(self, out, inp, stream=None):
        self.dist.all_to_all_single(out.reshape(-1), inp.reshape(-1), group=self.group)

    def all_gather(self, out, inp, stream=None):
        self.dist.all_gather_into_tensor(out.reshape(-1), inp.reshape(-1), group=self.group)

    def neighbor_exchange(self, send_first, send_last, recv_top, recv_bot, stream=None):
        """Spatial-split halo swap: my first row -> rank-1 (its bottom halo), my last
        row -> rank+1 (its top halo); global edges receive zeros."""
        d, r, g = self.dist, self.rank, self.world
        ops = []
        if r > 0:
            ops += [d.P2POp(d.isend, send_first.contiguous(), r - 1, self.group),
                    d.P2POp(d.irecv, recv_top, r - 1, self.group)]
        if r + 1 < g:
            ops += [d.P2POp(d.isend, send_last.contiguous(), r + 1, self.group),
                    d.P2POp(d.irecv, recv_bot, r + 1, self.group)]
        if ops:
            for w in d.batch_isend_irecv(ops):
                w.wait()
        if r == 0:
            recv_top.zero_()
        if r + 1 == g:
            recv_bot.zero_()


class _ThreadHub:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world


class ThreadComm:
    """g emulated ranks in one process (one thread each, same device): every
    rank synchronises its stream, publishes its send buffer, and after a
    barrier copies its own receive blocks; a second barrier keeps send buffers
    alive until every peer has copied. Kernels never wait on one another."""

    def __init__(self, hub, rank):
        self.hub, self.rank, self.world = hub, rank, hub.world

    @staticmethod
    def make(world):
        hub = _ThreadHub(world)
        return [ThreadComm(hub, r) for r in range(world)]

    def _exchange(self, out, inp, stream, pick):
        s = stream if stream is not None else torch.cuda.current_stream()
        s.synchronize()
        self.hub.slots[self.rank] = inp
        self.hub.barrier.wait()
        with torch.cuda.stream(s):
            pick(out)
        s.synchronize()
        self.hub.barrier.wait()

    def all_to_all(self, out, inp, stream=None):
        g = self.world

        def pick(o):
            ov = o.reshape(g, -1)
            for src in range(g):
                ov[src].copy_(self.hub.slots[src].reshape(g, -1)[self.rank])
        self._exchange(out, inp, stream, pick)

    def all_gather(self, out, inp, stream=None):
        g = self.world

        def pick(o):
            ov = o.reshape(g, -1)
            for src in range(g):
                ov[src].copy_(self.hub.slots[src].reshape(-1))
        self._exchange(out, inp, stream, pick)

    def neighbor_exchange(self, send_first, send_last, recv_top, recv_bot, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream()
        s.synchronize()
        self.hub.slots[self.rank] = (send_first, send_last)
        self.hub.barrier.wait()
        with torch.cuda.stream(s):
            if self.rank > 0:
                recv_top.copy_(self.hub.slots[self.rank - 1][1])
            else:
                recv_top.zero_()
            if self.rank + 1 < self.world:
                recv_bot.copy_(self.hub.slots[self.rank + 1][0])
            else:
                recv_bot.zero_()
        s.synchronize()
        self.hub.barrier.wait()
