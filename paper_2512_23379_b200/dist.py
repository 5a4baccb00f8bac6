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
state).

Two transports:
  * collective comms (`TorchComm`: NCCL all_to_all / all_gather through
    torch.distributed; `ThreadComm` emulates g ranks on one device for tests);
  * peer comms (`PeerComm`): the exchanges are FUSED into the producing kernels.
    Every rank exposes symmetric receive buffers; the QKV GEMM epilogue stores each
    head group's block straight into its owner's `qkv_recv`, the FMHA epilogue
    stores each output row into its owner's `ao`, and the out-projection epilogue
    replicates x0 into every rank's `x0tok`, all over NVLink peer mappings. One
    stream-ordered barrier after each producer replaces the collective. `IpcPeerComm`
    is the multi-process transport (cudaIpc handles exchanged through
    torch.distributed, device flag barrier); `ThreadPeerComm` runs g emulated ranks
    on one device (peer addresses are the other ranks' buffers, barrier on the host)
    so the fused layouts are tested without kernels that wait on one another.

Channels. A communicator's exchanges are ordered on ONE stream (its barrier epoch / collective
sequence). Work that runs concurrently on another stream or thread — the VAE decode on the
engine's decode stream, the host-side input broadcast of the ingest thread — takes its own
channel: `comm.channel(name)` (same transport, independent barrier flags and epoch, or its own
process group) and `comm.host_channel(name)` (host objects: `host_broadcast`). Channels are
created collectively (every rank, same order, from the main thread).
"""

import threading

import torch

from .errors import ConfigError


def slab_rows(h, world):
    """Row slab sizes of a spatial split of h rows over `world` ranks (first h % world ranks
    get one more row); the VAE decoder and the frame gather use the same partition."""
    if h < world:
        raise ConfigError("latent height %d cannot be split over %d ranks" % (h, world))
    return [h // world + (1 if i < h % world else 0) for i in range(world)]


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

    def channel(self, name):
        return self

    def host_channel(self, name):
        return self

    def host_broadcast(self, obj, src=0):
        return obj

    def gather_rows(self, full_name, full, slab, sizes, stream=None):
        full.copy_(slab)

    def all_gather_rows(self, full_name, full, slab, sizes, stream=None):
        full.copy_(slab)


def _on(stream):
    import contextlib
    if stream is None or not torch.cuda.is_available():
        return contextlib.nullcontext()
    return torch.cuda.stream(stream)


class TorchComm:
    """torch.distributed (NCCL on GPUs, gloo on CPU) equal-split collectives,
    enqueued on the caller's stream."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_to_all(self, out, inp, stream=None):
        with _on(stream):
            self.dist.all_to_all_single(out.reshape(-1), inp.reshape(-1), group=self.group)

    def all_gather(self, out, inp, stream=None):
        with _on(stream):
            self.dist.all_gather_into_tensor(out.reshape(-1), inp.reshape(-1), group=self.group)

    def channel(self, name):
        """Independent process group over the same ranks (collective: call on every rank)."""
        return TorchComm(self.dist.new_group(ranks=list(range(self.world))))

    def host_channel(self, name):
        """gloo group for host objects (the ingest thread's per-chunk input broadcast)."""
        return TorchComm(self.dist.new_group(ranks=list(range(self.world)), backend="gloo"))

    def host_broadcast(self, obj, src=0):
        lst = [obj]
        self.dist.broadcast_object_list(lst, src=src, group=self.group)
        return lst[0]

    def gather_rows(self, full_name, full, slab, sizes, stream=None):
        """Row slabs [T][rows_r][...] of every rank -> rank 0's full [T][sum(rows)][...]
        (slabs padded to the largest; only rank 0's `full` is written)."""
        mx = max(sizes)
        T, rows = slab.shape[0], slab.shape[1]
        with _on(stream):
            pad = torch.zeros((T, mx) + tuple(slab.shape[2:]), dtype=slab.dtype, device=slab.device)
            pad[:, :rows].copy_(slab)
            parts = [torch.empty_like(pad) for _ in range(self.world)]
            self.dist.all_gather(parts, pad, group=self.group)
            if self.rank == 0:
                r0 = 0
                for r, n in enumerate(sizes):
                    full[:, r0:r0 + n].copy_(parts[r][:, :n])
                    r0 += n

    def all_gather_rows(self, full_name, full, slab, sizes, stream=None):
        """gather_rows into EVERY rank's `full` (the decoder's mid attention needs every row's keys)."""
        mx = max(sizes)
        T, rows = slab.shape[0], slab.shape[1]
        with _on(stream):
            pad = torch.zeros((T, mx) + tuple(slab.shape[2:]), dtype=slab.dtype, device=slab.device)
            pad[:, :rows].copy_(slab)
            parts = [torch.empty_like(pad) for _ in range(self.world)]
            self.dist.all_gather(parts, pad, group=self.group)
            r0 = 0
            for r, n in enumerate(sizes):
                full[:, r0:r0 + n].copy_(parts[r][:, :n])
                r0 += n

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
        self.sym = {}
        self._subs = {}
        self._lock = threading.Lock()

    def sub(self, name):
        """The hub of channel `name` (created by whichever rank asks first)."""
        with self._lock:
            h = self._subs.get(name)
            if h is None:
                h = self._subs[name] = _ThreadHub(self.world)
            return h


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

    def channel(self, name):
        return ThreadComm(self.hub.sub(name), self.rank)

    def host_channel(self, name):
        return ThreadComm(self.hub.sub("host:" + name), self.rank)

    def host_broadcast(self, obj, src=0):
        if self.rank == src:
            self.hub.slots[src] = obj
        self.hub.barrier.wait()
        out = self.hub.slots[src]
        self.hub.barrier.wait()
        return out

    def gather_rows(self, full_name, full, slab, sizes, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream()
        s.synchronize()
        self.hub.slots[self.rank] = slab
        self.hub.barrier.wait()
        if self.rank == 0:
            with torch.cuda.stream(s):
                r0 = 0
                for r, n in enumerate(sizes):
                    full[:, r0:r0 + n].copy_(self.hub.slots[r])
                    r0 += n
            s.synchronize()
        self.hub.barrier.wait()

    def all_gather_rows(self, full_name, full, slab, sizes, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream()
        s.synchronize()
        self.hub.slots[self.rank] = slab
        self.hub.barrier.wait()
        with torch.cuda.stream(s):
            r0 = 0
            for r, n in enumerate(sizes):
                full[:, r0:r0 + n].copy_(self.hub.slots[r])
                r0 += n
        s.synchronize()
        self.hub.barrier.wait()

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


# ---------------------------------------------------------------- peer-memory transport
_TYPESTR = {torch.float32: "<f4", torch.int32: "<i4", torch.bfloat16: "<i2", torch.uint8: "|u1"}


class _SymAlloc:
    """Owner of one ftb_sym_alloc block, exposed to torch via __cuda_array_interface__
    (the tensor keeps this object alive; freeing it releases the block)."""

    def __init__(self, shape, dtype):
        import ctypes as C

        from . import _capi as A
        self.A = A
        n = 1
        for x in shape:
            n *= int(x)
        self.nbytes = max(1, n) * torch.tensor([], dtype=dtype).element_size()
        p = C.c_void_p()
        A.check(A.lib.ftb_sym_alloc(self.nbytes, C.byref(p)), "ftb_sym_alloc")
        self.ptr = p.value
        self.__cuda_array_interface__ = {"shape": tuple(int(x) for x in shape), "typestr": _TYPESTR[dtype],
                                         "data": (self.ptr, False), "version": 2, "strides": None}

    def __del__(self):
        try:
            self.A.lib.ftb_sym_free(self.ptr)
        except Exception:
            pass


def _sym_tensor(shape, dtype, device):
    own = _SymAlloc(shape, dtype)
    t = torch.as_tensor(own, device=device)
    return t.view(dtype) if dtype == torch.bfloat16 else t


class PeerComm:
    """Base of the fused-exchange transports. `sym(name, shape, dtype)` is collective
    (every rank calls it in the same order) and returns this rank's tensor;
    `addrs(name)` lists every rank's device address of that buffer (peer-mapped);
    `barrier(stream)` is stream-ordered: stores issued before it on any rank are
    visible to every rank's work enqueued after it."""

    peer = True
    capturable = False

    def __init__(self, world, rank):
        self.world, self.rank = int(world), int(rank)
        if self.world > 8:
            raise ConfigError("peer transport spans at most 8 ranks (one NVLink domain)")
        self._addrs = {}

    def addrs(self, name):
        return self._addrs[name]

    def halo_store(self, top_name, bot_name, offset_bytes, send_first, send_last, recv_top, recv_bot, stream=None):
        """Spatial-split halo swap over peer memory: my first rows go to rank-1's `bot_name`
        buffer and my last rows to rank+1's `top_name` buffer (byte offset `offset_bytes`),
        as device-to-device copies through the peer mappings; the global edges receive zeros.
        A barrier before the stores (the neighbours have finished the conv that read the
        previous halos) and one after (the rows are visible)."""
        s = stream if stream is not None else torch.cuda.current_stream()
        nb = send_first.numel() * send_first.element_size()
        self.barrier(s)
        with torch.cuda.stream(s):
            if self.rank > 0:
                _copy_to_peer(self._addrs[bot_name][self.rank - 1] + offset_bytes, send_first, nb, s)
            else:
                recv_top.zero_()
            if self.rank + 1 < self.world:
                _copy_to_peer(self._addrs[top_name][self.rank + 1] + offset_bytes, send_last, nb, s)
            else:
                recv_bot.zero_()
        self.barrier(s)

    def gather_rows(self, full_name, full, slab, sizes, stream=None):
        """Row slabs of every rank -> rank 0's symmetric buffer `full_name` ([T][H][...], H =
        sum(sizes)): each rank stores its slab rows straight into rank 0's frames over NVLink
        (one strided peer copy: T rows of rows*rowbytes), between two barriers (rank 0 has
        consumed the previous frames / the stores are visible)."""
        s = stream if stream is not None else torch.cuda.current_stream()
        T, rows = slab.shape[0], slab.shape[1]
        row_b = slab[0, 0].numel() * slab.element_size()
        H = sum(sizes)
        row0 = sum(sizes[:self.rank])
        self.barrier(s)
        _copy_2d_to_peer(self._addrs[full_name][0] + row0 * row_b, H * row_b, slab, rows * row_b, rows * row_b, T,
                         s)
        self.barrier(s)

    def all_gather_rows(self, full_name, full, slab, sizes, stream=None):
        """gather_rows into every rank's symmetric `full_name`: each rank stores its slab into all
        ranks' buffers at its row offset (one strided copy per destination), between two barriers."""
        s = stream if stream is not None else torch.cuda.current_stream()
        T, rows = slab.shape[0], slab.shape[1]
        row_b = slab[0, 0].numel() * slab.element_size()
        H = sum(sizes)
        row0 = sum(sizes[:self.rank])
        self.barrier(s)
        for dst in range(self.world):
            _copy_2d_to_peer(self._addrs[full_name][dst] + row0 * row_b, H * row_b, slab, rows * row_b, rows * row_b,
                             T, s)
        self.barrier(s)

    # collective fallbacks used outside the fused path (VAE halo, tests)
    def neighbor_exchange(self, send_first, send_last, recv_top, recv_bot, stream=None):
        raise NotImplementedError


def _copy_2d_to_peer(dst_addr, dpitch, src, spitch, width, height, stream):
    import ctypes as C
    from . import _capi as A
    A.call("ftb_copy_d2d_2d", C.c_void_p(int(dst_addr)), C.c_size_t(int(dpitch)), C.c_void_p(src.data_ptr()),
           C.c_size_t(int(spitch)), C.c_size_t(int(width)), C.c_size_t(int(height)), A.stream_ptr(stream))


def _copy_to_peer(dst_addr, src, nbytes, stream):
    """cudaMemcpyAsync D2D to a peer-mapped (or, emulated, same-device) address."""
    import ctypes as C
    from . import _capi as A
    A.call("ftb_copy_d2d", C.c_void_p(int(dst_addr)), C.c_void_p(src.data_ptr()), C.c_size_t(int(nbytes)),
           A.stream_ptr(stream))


class ThreadPeerComm(PeerComm):
    """g emulated ranks in one process (threads sharing one device): a rank's peer
    addresses are the other ranks' tensors; the barrier synchronises this rank's
    stream and meets the others on a host barrier (kernels never spin on peers)."""

    def __init__(self, hub, rank):
        super().__init__(hub.world, rank)
        self.hub = hub
        self._inner = ThreadComm(hub, rank)

    @staticmethod
    def make(world):
        hub = _ThreadHub(world)
        return [ThreadPeerComm(hub, r) for r in range(world)]

    def channel(self, name):
        return ThreadPeerComm(self.hub.sub(name), self.rank)

    def host_channel(self, name):
        return ThreadComm(self.hub.sub("host:" + name), self.rank)

    def sym(self, name, shape, dtype, device):
        t = torch.zeros(shape, dtype=dtype, device=device)
        torch.cuda.synchronize(device)
        self.hub.sym.setdefault(name, [None] * self.world)[self.rank] = t
        self.hub.barrier.wait()
        self._addrs[name] = [x.data_ptr() for x in self.hub.sym[name]]
        self.hub.barrier.wait()
        return t

    def barrier(self, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream()
        s.synchronize()
        self.hub.barrier.wait()

    def neighbor_exchange(self, *a, **k):
        self._inner.neighbor_exchange(*a, **k)


class IpcPeerComm(PeerComm):
    """One process per GPU of a node: buffers from ftb_sym_alloc, cudaIpc handles
    all-gathered through torch.distributed, imported once; barrier = ftb_peer_barrier
    (device flag words in a symmetric buffer, per-rank epoch counter on the device,
    so the whole chunk can be captured in a CUDA graph)."""

    def __init__(self, device, group=None, timeout_s=60.0, barrier_mode="device"):
        import torch.distributed as dist
        super().__init__(dist.get_world_size(group), dist.get_rank(group))
        if barrier_mode not in ("device", "host"):
            raise ConfigError("barrier_mode must be 'device' or 'host'")
        self.dist, self.group, self.device, self.timeout_s = dist, group, device, float(timeout_s)
        # "host": stream sync + process-group barrier (tests that put several ranks on one
        # GPU, where a spinning kernel must never wait on another process's kernel)
        self.barrier_mode = barrier_mode
        self.capturable = barrier_mode == "device"
        self._coll = TorchComm(group)
        self._imported = []
        self._keep = []
        self.flags = self.sym("__flags", (self.world,), torch.int32, device)
        self.epoch = torch.zeros(1, dtype=torch.int32, device=device)

    def sym(self, name, shape, dtype, device=None):
        import ctypes as C

        from . import _capi as A
        t = _sym_tensor(shape, dtype, device or self.device)
        self._keep.append(t)
        h = C.create_string_buffer(A.IPC_HANDLE_BYTES)
        A.check(A.lib.ftb_ipc_export(t.data_ptr(), h), "ftb_ipc_export")
        handles = [None] * self.world
        self.dist.all_gather_object(handles, bytes(h.raw), group=self.group)
        addrs = []
        for r, hb in enumerate(handles):
            if r == self.rank:
                addrs.append(t.data_ptr())
                continue
            p = C.c_void_p()
            A.check(A.lib.ftb_ipc_import(C.create_string_buffer(hb, A.IPC_HANDLE_BYTES), C.byref(p)),
                    "ftb_ipc_import")
            self._imported.append(p.value)
            addrs.append(p.value)
        self._addrs[name] = addrs
        return t

    def barrier(self, stream=None):
        from . import ops
        if self.barrier_mode == "host":
            (stream if stream is not None else torch.cuda.current_stream()).synchronize()
            self.dist.barrier(group=self.group)
            return
        ops.peer_barrier(self._addrs["__flags"], self.epoch, self.rank, self.world, self.timeout_s, stream=stream)

    def neighbor_exchange(self, *a, **k):
        self._coll.neighbor_exchange(*a, **k)

    def channel(self, name):
        """Same ranks, own process group, own flag words and epoch counter (a barrier stream of
        its own: the engine's decode stream runs the VAE halo barriers concurrently with the
        DiT barriers on the denoise stream)."""
        grp = self.dist.new_group(ranks=list(range(self.world)))
        return IpcPeerComm(self.device, group=grp, timeout_s=self.timeout_s, barrier_mode=self.barrier_mode)

    def host_channel(self, name):
        return TorchComm(self.dist.new_group(ranks=list(range(self.world)), backend="gloo"))

    def close(self):
        from . import _capi as A
        for p in self._imported:
            A.lib.ftb_ipc_close(p)
        self._imported = []
