"""Torch-tensor plumbing over the C-ABI: device buffers in, device buffers out.

torch is used only to own device memory and streams; all arithmetic happens
in the sm_100a kernels behind libhetplan_b200.so (capi.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import torch

from . import capi
from .capi import check, lib

GROUP = 128


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream: torch.cuda.Stream | None) -> int | None:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream or None


@dataclass
class QuantizedWeight:
    """Packed adaptive-bitwidth weight of one linear op (hp_qweight)."""

    n_out: int
    k_in: int
    bits: int
    scheme: int
    packed: torch.Tensor
    scale: torch.Tensor | None
    zero: torch.Tensor | None
    _c: capi.hp_qweight = field(init=False, repr=False)

    def __post_init__(self):
        self._c = capi.hp_qweight(self.n_out, self.k_in, self.bits, self.scheme,
                                  self.packed.data_ptr(), _ptr(self.scale), _ptr(self.zero))

    @property
    def c(self) -> capi.hp_qweight:
        return self._c

    @property
    def nbytes(self) -> int:
        n = self.packed.numel()
        if self.scale is not None:
            n += self.scale.numel() * 4
        if self.zero is not None:
            n += self.zero.numel() * 4
        return n


def packed_bytes(n_out: int, k_in: int, bits: int) -> int:
    return int(lib.hp_packed_bytes(n_out, k_in, bits))


def quantize(w: torch.Tensor, bits: int, scheme: int = capi.HP_SYMMETRIC,
             rounding: int = capi.HP_NEAREST, want_fp64: bool = False,
             stream: torch.cuda.Stream | None = None, stats: torch.Tensor | None = None):
    """K1: group-wise quantize + pack a bf16 [n_out, k_in] CUDA tensor.

    Returns QuantizedWeight, plus (step64, zero64) [n_out, G] fp64 tensors
    when want_fp64 is set (the reference's per-group step / grid origin).
    stats: optional device fp64[5]; K1's pass also writes the indicator's
    weight statistics into stats[0..2] (hp_quant_pack_stats).
    """
    assert w.dtype == torch.bfloat16 and w.is_cuda and w.dim() == 2
    n_out, k_in = w.shape
    ldw = w.stride(0)
    assert w.stride(1) == 1
    dev = w.device
    nbytes = packed_bytes(n_out, k_in, bits)
    if nbytes < 0:
        raise capi.InvalidArgument(capi.HP_EINVAL, f"quantize: unsupported bits={bits} or shape")
    packed = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    nsc = int(lib.hp_scale_count(n_out, k_in))
    scale = torch.empty(nsc, dtype=torch.float32, device=dev) if bits != 16 else None
    zero = (torch.empty(nsc, dtype=torch.float32, device=dev)
            if bits != 16 and scheme == capi.HP_ASYMMETRIC else None)
    step64 = zero64 = None
    if want_fp64 and bits != 16:
        G = -(-k_in // GROUP)
        step64 = torch.empty(n_out, G, dtype=torch.float64, device=dev)
        zero64 = torch.empty(n_out, G, dtype=torch.float64, device=dev)
    if stats is not None:
        assert stats.dtype == torch.float64 and stats.numel() >= 5 and stats.device == dev
        check(lib.hp_quant_pack_stats(w.data_ptr(), n_out, k_in, ldw, bits, scheme, rounding,
                                      packed.data_ptr(), _ptr(scale), _ptr(zero), _ptr(step64),
                                      _ptr(zero64), stats.data_ptr(), _stream(stream)))
    else:
        check(lib.hp_quant_pack(w.data_ptr(), n_out, k_in, ldw, bits, scheme, rounding,
                                packed.data_ptr(), _ptr(scale), _ptr(zero), _ptr(step64),
                                _ptr(zero64), _stream(stream)))
    qw = QuantizedWeight(n_out, k_in, bits, scheme, packed, scale, zero)
    if want_fp64:
        return qw, step64, zero64
    return qw


def unpack(qw: QuantizedWeight, stream=None):
    """Stored codes [n_out, k_in] (u8; int16 view of bf16 words for 16-bit),
    and row-major fp32 scale / zero [n_out, G]."""
    G = -(-qw.k_in // GROUP)
    dev = qw.packed.device
    if qw.bits == 16:
        codes = torch.empty(qw.n_out, qw.k_in, dtype=torch.int16, device=dev)
    else:
        codes = torch.empty(qw.n_out, qw.k_in, dtype=torch.uint8, device=dev)
    scale = torch.empty(qw.n_out, G, dtype=torch.float32, device=dev) if qw.scale is not None else None
    zero = torch.empty(qw.n_out, G, dtype=torch.float32, device=dev) if qw.zero is not None else None
    check(lib.hp_quant_unpack(C.byref(qw.c), codes.data_ptr(), _ptr(scale), _ptr(zero),
                              _stream(stream)))
    return codes, scale, zero


def dequant(qw: QuantizedWeight, stream=None) -> torch.Tensor:
    out = torch.empty(qw.n_out, qw.k_in, dtype=torch.bfloat16, device=qw.packed.device)
    check(lib.hp_dequant(C.byref(qw.c), out.data_ptr(), _stream(stream)))
    return out


def indicator_stats(w: torch.Tensor | None, x: torch.Tensor | None, stream=None,
                    out: torch.Tensor | None = None) -> torch.Tensor:
    """K2: device fp64[5] = {d_w, w_min, w_max, x_mean, x_var}.

    w=None: only the calibration part [3..4] is written into `out` (whose
    [0..2] came from quantize(..., stats=out), K1's fused weight pass)."""
    assert w is not None or (x is not None and out is not None)
    n_out, k_in = w.shape if w is not None else (0, x.shape[1])
    dev = (w if w is not None else x).device
    if out is None:
        out = torch.empty(5, dtype=torch.float64, device=dev)
    tokens = 0 if x is None else x.shape[0]
    ldx = 0 if x is None else x.stride(0)
    check(lib.hp_indicator_stats(_ptr(w), n_out, k_in, 0 if w is None else w.stride(0), _ptr(x),
                                 tokens, ldx, out.data_ptr(), _stream(stream)))
    return out


class Workspace:
    """Grow-only split-K workspace (zeroed once; kernels leave it zeroed)."""

    def __init__(self, device):
        self.device = device
        self.buf = torch.zeros(0, dtype=torch.uint8, device=device)

    def get(self, nbytes: int) -> torch.Tensor:
        if nbytes > self.buf.numel():
            self.buf = torch.zeros(max(nbytes, 2 * self.buf.numel()), dtype=torch.uint8,
                                   device=self.device)
        return self.buf


_ws: dict = {}


def workspace_for(device) -> Workspace:
    key = str(device)
    if key not in _ws:
        _ws[key] = Workspace(device)
    return _ws[key]


def qlinear(qw: QuantizedWeight, x: torch.Tensor, phase: int = capi.HP_DECODE,
            out: torch.Tensor | None = None, residual: torch.Tensor | None = None,
            relu: bool = False, stream=None, workspace: Workspace | None = None) -> torch.Tensor:
    """K3 (decode) / K4 (prefill): out = epi(x @ dequant(W).T) (+ residual)."""
    assert x.dtype == torch.bfloat16 and x.is_cuda and x.stride(-1) == 1
    m = x.shape[0]
    if out is None:
        out = torch.empty(m, qw.n_out, dtype=torch.bfloat16, device=x.device)
    ws = workspace or workspace_for(x.device)
    need = int(lib.hp_qlinear_workspace_bytes(C.byref(qw.c), m, phase))
    buf = ws.get(need) if need else None
    check(lib.hp_qlinear(C.byref(qw.c), x.data_ptr(), x.stride(0), m, out.data_ptr(),
                         out.stride(0), _ptr(residual),
                         residual.stride(0) if residual is not None else 0,
                         capi.HP_EPI_RELU if relu else capi.HP_EPI_NONE, phase,
                         _ptr(buf), need, _stream(stream)))
    return out


# ---- decoder glue (decoder.cu; hp_embed / hp_attention_* / hp_argmax) ----
def embed(tok: torch.Tensor, E: torch.Tensor, P: torch.Tensor | None, pos0: int,
          pos_per_req: bool = False, s_tokens: int = 1, stream=None) -> torch.Tensor:
    """x[r] = E[tok[r]] + P[pos(r) + 2] (OPT learned positions)."""
    rows = tok.numel()
    h = E.shape[1]
    x = torch.empty(rows, h, dtype=torch.bfloat16, device=E.device)
    check(lib.hp_embed(tok.data_ptr(), rows, pos0, int(pos_per_req), s_tokens, E.data_ptr(),
                       _ptr(P), P.shape[0] if P is not None else 0, h, E.shape[0], x.data_ptr(),
                       _stream(stream)))
    return x


def attention_prefill(qkv: torch.Tensor, reqs: int, s: int, hd: int, kc: torch.Tensor,
                      vc: torch.Tensor, req0: int, s_max: int, stream=None) -> torch.Tensor:
    h = qkv.shape[1] // 3
    out = torch.empty(reqs * s, h, dtype=torch.bfloat16, device=qkv.device)
    check(lib.hp_attention_prefill(qkv.data_ptr(), reqs, s, h, hd, out.data_ptr(), kc.data_ptr(),
                                   vc.data_ptr(), req0, s_max, _stream(stream)))
    return out


_attn_ws: dict = {}


def attention_decode(qkv: torch.Tensor, hd: int, p: int, kc: torch.Tensor, vc: torch.Tensor,
                     req0: int, s_max: int, split: int = 1, stream=None) -> torch.Tensor:
    rows, h = qkv.shape[0], qkv.shape[1] // 3
    out = torch.empty(rows, h, dtype=torch.bfloat16, device=qkv.device)
    need = int(lib.hp_attention_decode_workspace_bytes(rows, h, hd, split))
    ws = None
    if need:
        key = str(qkv.device)
        if key not in _attn_ws or _attn_ws[key].numel() < need:
            _attn_ws[key] = torch.zeros(need, dtype=torch.uint8, device=qkv.device)
        ws = _attn_ws[key]
    check(lib.hp_attention_decode(qkv.data_ptr(), rows, h, hd, p, out.data_ptr(), kc.data_ptr(),
                                  vc.data_ptr(), req0, s_max, split, _ptr(ws), need, _stream(stream)))
    return out


def argmax(logits: torch.Tensor, stream=None) -> torch.Tensor:
    rows, vocab = logits.shape
    tok = torch.empty(rows, dtype=torch.int32, device=logits.device)
    check(lib.hp_argmax(logits.data_ptr(), logits.stride(0), rows, vocab, tok.data_ptr(),
                        _stream(stream)))
    return tok
