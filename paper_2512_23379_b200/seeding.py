"""Deterministic RNG stream derivation (host side).

Same contract as the reference's `rng_for` (`pkg/src/ftlk/seeding.py:26-36`):
a PCG64 generator keyed by the flattened (seed, *tags) path through
`numpy.random.SeedSequence`. The per-chunk initial noise of the sampler is
drawn here on the host so it is bit-identical to the reference
(`pkg/src/ftlk/streaming.py:293`, `pkg/src/ftlk/diffusion.py:225`), then
uploaded once per chunk.
"""

import numpy as np

# Tag values are part of the reproducibility contract (seeding.py:12-21).
SIGNAL = 1
DYNAMICS = 2
IDENTITY = 3
INIT = 4
DATA = 5
TRAIN = 6
ROLLOUT = 7
DMD = 8
STREAM_NOISE = 9
EVAL = 10

_MASK64 = (1 << 64) - 1


def flatten_path(parts):
    out = []
    stack = [iter(parts)]
    while stack:
        try:
            item = next(stack[-1])
        except StopIteration:
            stack.pop()
            continue
        if isinstance(item, (tuple, list)):
            stack.append(iter(item))
        else:
            out.append(int(item) & _MASK64)
    return out


def rng_for(seed, *tags) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(flatten_path((seed,) + tags))))


def chunk_noise(seed, chunk_index: int, shape) -> np.ndarray:
    """Initial sampler state of chunk `chunk_index`: standard normal f64 of
    `shape` from stream (seed, STREAM_NOISE, c), C order."""
    return rng_for(seed, STREAM_NOISE, chunk_index).standard_normal(tuple(shape))
