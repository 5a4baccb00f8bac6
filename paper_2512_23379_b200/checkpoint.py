"""FTLK checkpoint I/O (reference format `pkg/src/ftlk/checkpoint.py:1-103`) and a
streaming loader into bf16 device weights.

Container (little-endian): b"FTLK", u32 version=1, u32 count, then per tensor
u16 name length, UTF-8 name, u8 rank, u32 dims[rank], float64 data; then a
u32-length canonical JSON trailer {"net": {...}, "role": ...} (sorted keys,
no whitespace). `load` is strict in the reference's way (magic, version,
truncation, duplicate names, trailing bytes, names/shapes vs the declared
NetConfig) and raises ConfigError. `save` is canonical, so an unmodified
store round-trips byte for byte.

`load_device_weights` walks the file once and uploads each tensor as it is
parsed (bf16 W^T / fp32 vectors), so a 14B-shape checkpoint never needs its
105 GiB float64 image on the host.
"""

import dataclasses
import json
import mmap
import struct

import numpy as np

from .config import NetConfig, param_shapes
from .errors import ConfigError
from .net import ParamStore

MAGIC = b"FTLK"
VERSION = 1
ROLES = ("teacher_real", "generator_student", "fake_score")


def _net_json(net: NetConfig) -> dict:
    d = dataclasses.asdict(net)
    # reference-shaped configs stay byte-identical to the reference writer
    if net.mode == "ftlk":
        d = {k: d[k] for k in ("model_dim", "layers", "heads", "ff_dim", "latent_dim")}
    else:
        d["patch"] = list(d["patch"])
    return d


def save(path, store: ParamStore, role: str, net: NetConfig) -> None:
    if role not in ROLES:
        raise ConfigError("unknown checkpoint role %r" % (role,))
    parts = [MAGIC, struct.pack("<II", VERSION, len(store.params))]
    for name, arr in store.params.items():
        a = np.ascontiguousarray(arr, dtype="<f8")
        nb = name.encode("utf-8")
        parts.append(struct.pack("<H", len(nb)) + nb + struct.pack("<B", a.ndim))
        parts.append(struct.pack("<%dI" % a.ndim, *a.shape))
        parts.append(a.tobytes())
    trailer = json.dumps({"role": role, "net": _net_json(net)}, sort_keys=True, separators=(",", ":")).encode()
    parts.append(struct.pack("<I", len(trailer)) + trailer)
    with open(path, "wb") as f:
        f.write(b"".join(parts))


class _Reader:
    def __init__(self, buf, path):
        self.buf, self.off, self.path = buf, 0, path

    def take(self, n):
        if self.off + n > len(self.buf):
            raise ConfigError("truncated checkpoint %s" % self.path)
        v = self.buf[self.off:self.off + n]
        self.off += n
        return v

    def unpack(self, fmt):
        return struct.unpack(fmt, self.take(struct.calcsize(fmt)))


def _entries(buf, path):
    """Yields (name, ndarray view) then returns via StopIteration value the trailer."""
    r = _Reader(buf, path)
    if bytes(r.take(4)) != MAGIC:
        raise ConfigError("%s is not an FTLK checkpoint (bad magic)" % path)
    (version,) = r.unpack("<I")
    if version != VERSION:
        raise ConfigError("unsupported checkpoint version %d" % version)
    (count,) = r.unpack("<I")
    seen = set()
    for _ in range(count):
        (nlen,) = r.unpack("<H")
        name = bytes(r.take(nlen)).decode("utf-8")
        (rank,) = r.unpack("<B")
        dims = r.unpack("<%dI" % rank) if rank else ()
        size = int(np.prod(dims)) if rank else 1
        if name in seen:
            raise ConfigError("duplicate tensor name %r in %s" % (name, path))
        seen.add(name)
        yield name, np.frombuffer(r.take(8 * size), dtype="<f8").reshape(dims)
    (tlen,) = r.unpack("<I")
    meta = json.loads(bytes(r.take(tlen)).decode("utf-8"))
    if r.off != len(buf):
        raise ConfigError("%s has %d trailing bytes" % (path, len(buf) - r.off))
    return meta


def _check(names_shapes, meta):
    role = meta.get("role")
    if role not in ROLES:
        raise ConfigError("unknown checkpoint role %r" % (role,))
    netd = dict(meta["net"])
    if "patch" in netd:
        netd["patch"] = tuple(netd["patch"])
    net = NetConfig(**netd)
    want = [(n, tuple(s)) for n, s in param_shapes(net)]
    if [n for n, _ in names_shapes] != [n for n, _ in want]:
        raise ConfigError("checkpoint tensors do not match the declared net config")
    for (n, s), (_, ws) in zip(names_shapes, want):
        if tuple(s) != ws:
            raise ConfigError("tensor %r has shape %s, want %s" % (n, tuple(s), ws))
    return role, net


def load(path):
    """Returns (ParamStore, role, NetConfig) — reference `checkpoint.load` contract."""
    with open(path, "rb") as f:
        buf = f.read()
    params = {}
    gen = _entries(memoryview(buf), path)
    while True:
        try:
            name, arr = next(gen)
        except StopIteration as stop:
            meta = stop.value
            break
        params[name] = np.array(arr, dtype=np.float64)
    role, net = _check([(n, a.shape) for n, a in params.items()], meta)
    return ParamStore(params), role, net


def load_device_weights(path, device="cuda"):
    """Stream a checkpoint into bf16 device weights (model.DeviceWeights) one
    tensor at a time. Returns (DeviceWeights, role, NetConfig). A malformed file
    raises ConfigError (the mapping is closed first)."""
    with open(path, "rb") as f:
        mm = mmap.mmap(f.fileno(), 0, access=mmap.ACCESS_READ)
    failure = None
    try:
        return _device_weights_from(mm, path, device)
    except BaseException as e:  # noqa: BLE001
        # the loader's frames (kept alive by the traceback) still export views of the mapping,
        # and mm.close() would raise BufferError over the real error: drop them first
        e.__traceback__ = None
        failure = e
    finally:
        mm.close()
    raise failure


def _device_weights_from(mm, path, device):
    import torch

    from .model import DeviceWeights, round8
    view = memoryview(mm)
    # first pass: trailer + shape validation without materialising data
    gen = _entries(view, path)
    shapes = []
    while True:
        try:
            name, arr = next(gen)
        except StopIteration as stop:
            meta = stop.value
            break
        shapes.append((name, arr.shape))
        del arr
    role, net = _check(shapes, meta)
    w = DeviceWeights(net, device)
    gen = _entries(view, path)
    for name, arr in gen:
        if arr.ndim == 2 and not name.endswith(".mod"):
            K, N = arr.shape
            wt = torch.zeros(N, round8(K), dtype=torch.bfloat16, device=w.device)
            wt[:, :K] = torch.from_numpy(np.array(arr.T)).to(w.device).to(torch.bfloat16)
            w.mats[name] = (wt, K)
        else:
            w.vecs[name] = torch.from_numpy(np.array(arr)).to(torch.float32).to(w.device)
        del arr
    w._fuse()
    del gen
    view.release()
    return w, role, net
