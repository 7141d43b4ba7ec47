"""Shared helpers for tests (bf16 bit handling)."""
import numpy as np


def to_bf16_bits(a) -> np.ndarray:
    f = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounding = ((f >> 16) & 1) + 0x7FFF
    return ((f + rounding) >> 16).astype(np.uint16)


def bf16_bits_to_f64(b) -> np.ndarray:
    return (np.asarray(b).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def bits_to_torch(b, device):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(b).view(np.int16).copy())
    return t.view(torch.bfloat16).to(device)


def torch_to_bits(t) -> np.ndarray:
    import torch
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
