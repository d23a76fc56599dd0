"""Seeded synthetic inputs shared by the oracle tests, the CUDA path and bench.py.

This module holds NO arithmetic of the AutoChunk method: it only draws random
numbers and encodes them in the storage format a graph declares.  Both sides
(oracle/ and paper_2401_10652_b200/) consume its output; neither imports the
other.  Recipe (SURVEY.md §8(d) "Synthetic inputs"):

* RNG: numpy Generator(PCG64(seed)); weights use seed 1234 + weight index,
  activations use seed 42 + input index.
* Values are drawn in fp32; bf16 tensors are then rounded to bf16 with
  round-to-nearest-even and the SAME bits are uploaded to the GPU.
* x, z ~ N(0,1); matrix weights ~ N(0, 1/fan_in); biases ~ N(0, 0.02^2);
  LayerNorm gamma ~ 1 + N(0, 0.02^2), beta ~ N(0, 0.02^2).
"""
from __future__ import annotations

import numpy as np

WEIGHT_SEED = 1234
ACT_SEED = 42

ROLES = ("act", "matrix", "bias", "ln_gamma", "ln_beta")


def bf16_bits(a: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit patterns (uint16), round-to-nearest-even (finite inputs)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    """bf16 bit patterns -> exact fp32 values."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def draw(shape, role: str, fan_in: int, seed: int) -> np.ndarray:
    """Draw one fp32 tensor of the given role (no rounding)."""
    if role not in ROLES:
        raise ValueError(f"unknown role {role!r}")
    rng = np.random.Generator(np.random.PCG64(seed))
    shape = tuple(int(s) for s in shape)
    if role == "act":
        v = rng.standard_normal(shape, dtype=np.float32)
    elif role == "matrix":
        v = rng.standard_normal(shape, dtype=np.float32) * np.float32(1.0 / np.sqrt(max(fan_in, 1)))
    elif role == "bias" or role == "ln_beta":
        v = rng.standard_normal(shape, dtype=np.float32) * np.float32(0.02)
    else:  # ln_gamma
        v = np.float32(1.0) + rng.standard_normal(shape, dtype=np.float32) * np.float32(0.02)
    return v.astype(np.float32)


class Sample:
    """One generated tensor: `value` is the exact stored value as float64,
    `storage` is what gets uploaded (uint16 bf16 bits, float32 or float64)."""

    __slots__ = ("tid", "dtype", "shape", "storage", "value")

    def __init__(self, tid, dtype, shape, storage, value):
        self.tid, self.dtype, self.shape, self.storage, self.value = tid, dtype, shape, storage, value


def encode(v32: np.ndarray, dtype: str):
    if dtype == "bf16":
        bits = bf16_bits(v32)
        return bits, bf16_bits_to_f32(bits).astype(np.float64)
    if dtype == "f32":
        return v32, v32.astype(np.float64)
    if dtype == "f64":
        return v32.astype(np.float64), v32.astype(np.float64)
    raise ValueError(dtype)


def make_inputs(specs, scale_seed: int = 0):
    """specs: list of (tid, kind ∈ {input, weight}, dtype, shape, role, fan_in), in
    graph declaration order.  Returns {tid: Sample}.  Weight i uses seed
    1234 + i, input i uses seed 42 + i (+ scale_seed for test variations)."""
    out = {}
    wi = ii = 0
    for tid, kind, dtype, shape, role, fan_in in specs:
        if kind == "weight":
            seed = WEIGHT_SEED + wi + scale_seed
            wi += 1
        else:
            seed = ACT_SEED + ii + scale_seed
            ii += 1
        v32 = draw(shape, role, fan_in, seed)
        storage, value = encode(v32, dtype)
        out[tid] = Sample(tid, dtype, tuple(shape), storage, value)
    return out
