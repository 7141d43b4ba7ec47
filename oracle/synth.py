"""ORACLE / TEST INFRASTRUCTURE: bit-reproducible synthetic tensors.

Mirror of the product's device initialiser (paper_2403_01136_b200/csrc/
glue.cu, hp_synth_bf16): element i of a tensor with seed S is
    r1 = splitmix64(S ^ 2i), r2 = splitmix64(S ^ (2i+1))
    v  = (lo32(r1) + hi32(r1) + lo32(r2) + hi32(r2)) - 2^33   (Irwin-Hall(4))
    w  = bf16_rne( float32( mean + v * (std * sqrt(3) * 2^-32) ) )
All steps are exact integer ops or single IEEE roundings, so numpy here and
CUDA on the GPU produce identical bits.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
SQRT3_2M32 = 1.7320508075688772 * 2.3283064365386963e-10


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def seed_for(*parts: int, base: int = 2403) -> int:
    s = np.uint64(base)
    for p in parts:
        s = splitmix64(np.array([s ^ np.uint64(p)], dtype=np.uint64))[0]
    return int(s)


def synth_bits(n: int, seed: int, mean: float, std: float) -> np.ndarray:
    """uint16 bf16 bit patterns of n synthetic values."""
    i = np.arange(n, dtype=np.uint64)
    s = np.uint64(seed)
    r1 = splitmix64(s ^ (i << np.uint64(1)))
    r2 = splitmix64(s ^ ((i << np.uint64(1)) | np.uint64(1)))
    lo = np.uint64(0xFFFFFFFF)
    tot = (r1 & lo) + (r1 >> np.uint64(32)) + (r2 & lo) + (r2 >> np.uint64(32))
    v = (tot.astype(np.int64) - (1 << 33)).astype(np.float64)
    scale = std * SQRT3_2M32
    w = (mean + v * scale).astype(np.float32)
    f = w.view(np.uint32).astype(np.uint64)
    return ((f + ((f >> np.uint64(16)) & np.uint64(1)) + np.uint64(0x7FFF)) >> np.uint64(16)).astype(np.uint16)


def synth_tokens(n: int, seed: int, vocab: int) -> np.ndarray:
    """int32 token ids: splitmix64(seed ^ i) % vocab (mirror of the runtime's
    synth_tokens_kernel, csrc/decoder.cu)."""
    i = np.arange(n, dtype=np.uint64)
    return (splitmix64(np.uint64(seed) ^ i) % np.uint64(vocab)).astype(np.int32)
