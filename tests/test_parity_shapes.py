"""Oracle parity at the BENCHED and TARGET op shapes.

Every op of the OPT-13B (bench, BASELINE configs[1]) and OPT-30B
(north_star target) decoder layer -- qkv [3h1 x h1], out [h1 x h1],
fc1 [h2 x h1], fc2 [h1 x h2] -- at 3/4/8/16 bits x {asym, sym} (and of the
OPT-66B / BLOOM-176B layers, configs[3..4], at 3 asym / 4, 8, 16 sym), through
K3 (decode, m = xi = 32, stream-K) and K4 (prefill, m = eta*s = 2048; out /
fc2 take the stream-K prefill split there), against the CPU oracle:

  * K1: the sampled rows' codes and fp64 steps/zeros are bit-exact against
    oracle/hp_oracle.c's restatement of quantize() (indicator.cpp:19-56),
    which tests/test_oracle.py pins to the reference's own compiled code;
  * K3/K4: y[:, rows] against the oracle's fp64 GEMM over the ORACLE's
    dequantized weights zero + (code - off) * step (indicator.cpp:53) --
    nothing from the library feeds the reference side.

Rows are sampled (64 per op, always including the first and last row and a
row of every 128-row tile boundary the sample hits) so the fp64 CPU GEMM
stays within seconds; every token column is checked. Tolerance: the
north_star's normwise max|y - y_ref| / max|y_ref| <= 1e-2 (bf16 output,
fp32 accumulation); we assert the tighter 8e-3.

K1 at production sizes (full matrices, not sampled): OPT-13B fc1
[20480 x 5120], OPT-30B fc1 [28672 x 7168] and BLOOM-176B fc1
[57344 x 14336] (822M weights), every code bit-exact against the oracle.
"""
import zlib

import numpy as np
import pytest

from tests.util import bf16_bits_to_f64, torch_to_bits

pytestmark = pytest.mark.gpu

# tighter than the north_star's 1e-2; the observed error of every case is
# printed (-rA). Before the centred asymmetric operand (layout.cuh
# asym_base2) asymmetric 3/4-bit OPT-30B qkv/out reached 1.01e-2.
TOL = 8e-3
MODELS = {"opt13b": (5120, 20480), "opt30b": (7168, 28672)}
OPS = {"qkv": lambda h1, h2: (3 * h1, h1), "out": lambda h1, h2: (h1, h1),
       "fc1": lambda h1, h2: (h2, h1), "fc2": lambda h1, h2: (h1, h2)}
BITS_SCHEMES = [(3, 0), (3, 1), (4, 0), (4, 1), (8, 0), (8, 1), (16, 1)]
M_PHASE = [(32, 1), (2048, 0)]  # K3 decode (xi = 32), K4 prefill (eta*s = 4*512)


def _weights(n, k, seed, dev):
    import torch
    g = torch.Generator(device=dev).manual_seed(seed)
    w = torch.randn(n, k, generator=g, device=dev) * 0.02
    # 0.1% x8 outliers: exercise range and clamp
    mask = torch.rand(n, k, generator=g, device=dev) < 1e-3
    w = torch.where(mask, w * 8, w)
    return w.to(torch.bfloat16)


def _rows(n, rng, count=64):
    r = set(rng.choice(n, size=min(count, n) - 2, replace=False).tolist()) | {0, n - 1}
    return np.array(sorted(r), dtype=np.int64)


def _err(got, ref):
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))


# configs[3] / configs[4] layer shapes (OPT-66B, BLOOM-176B; their 8-stage
# plans use 3/4/8/16 bits): one bit width per scheme family, every op
MODELS_BIG = {"opt66b": (9216, 36864), "bloom176b": (14336, 57344)}
BITS_SCHEMES_BIG = [(3, 0), (4, 1), (8, 1), (16, 1)]
CASES = ([(m, b, s) for m in MODELS for b, s in BITS_SCHEMES] +
         [(m, b, s) for m in MODELS_BIG for b, s in BITS_SCHEMES_BIG])


@pytest.mark.parametrize("model,bits,scheme", CASES, ids=[f"{m}-b{b}s{s}" for m, b, s in CASES])
@pytest.mark.parametrize("op", list(OPS))
def test_benched_shape_k1_k3_k4_vs_oracle(cuda, model, op, bits, scheme):
    import torch

    import oracle
    from paper_2403_01136_b200 import qweight
    h1, h2 = {**MODELS, **MODELS_BIG}[model]
    n, k = OPS[op](h1, h2)
    seed = zlib.crc32(f"{model}/{op}/{bits}/{scheme}".encode()) % 2**31
    rng = np.random.default_rng(seed)
    w = _weights(n, k, seed, cuda)
    rows = _rows(n, rng)
    wb_rows = torch_to_bits(w[torch.from_numpy(rows).to(cuda)])
    port = oracle.port()
    if bits == 16:
        o_codes, o_step, o_zero = wb_rows, None, None
        qw = qweight.quantize(w, 16)
        codes, _, _ = qweight.unpack(qw)
        got_rows = codes[torch.from_numpy(rows).to(cuda)].cpu().numpy().view(np.uint16)
        np.testing.assert_array_equal(got_rows, o_codes)
    else:
        qw, step64, zero64 = qweight.quantize(w, bits, scheme, want_fp64=True)
        o_codes, o_step, o_zero = port.quantize_matrix(wb_rows, bits, scheme)
        codes, _, _ = qweight.unpack(qw)
        idx = torch.from_numpy(rows).to(cuda)
        # K1 parity on the sampled rows: codes, fp64 step and grid origin
        np.testing.assert_array_equal(codes[idx].cpu().numpy(), o_codes)
        np.testing.assert_array_equal(step64[idx].cpu().numpy().view(np.uint64),
                                      o_step.view(np.uint64))
        np.testing.assert_array_equal(zero64[idx].cpu().numpy() + 0.0, o_zero + 0.0)
    del codes
    for m, phase in M_PHASE:
        x = (torch.randn(m, k, generator=torch.Generator(device=cuda).manual_seed(seed + m),
                         device=cuda) + 0.05).to(torch.bfloat16)
        y = qweight.qlinear(qw, x, phase=phase)
        got = bf16_bits_to_f64(torch_to_bits(y[:, torch.from_numpy(rows).to(cuda)]))
        ref = port.qlinear(torch_to_bits(x), o_codes, o_step, o_zero, bits, scheme)
        e = _err(got, ref.astype(np.float64))
        print(f"PARITY {model} {op} b{bits} s{scheme} m={m} err={e:.3e}")
        assert e <= TOL, f"{model} {op} [{n}x{k}] b{bits} s{scheme} m={m}: normwise err {e}"
        # run-to-run determinism of the stream-K / persistent split
        assert torch.equal(y, qweight.qlinear(qw, x, phase=phase))


@pytest.mark.parametrize("shape", [(20480, 5120), (28672, 7168), (57344, 14336)],
                         ids=["opt13b_fc1", "opt30b_fc1", "bloom176b_fc1"])
@pytest.mark.parametrize("bits,scheme", [(3, 1), (4, 0), (8, 1)])
def test_k1_production_size_bit_exact(cuda, shape, bits, scheme):
    """Every code / fp64 step / zero of a full production-size op vs the oracle."""
    import torch

    import oracle
    from paper_2403_01136_b200 import qweight
    n, k = shape
    w = _weights(n, k, n + bits + scheme, cuda)
    qw, step64, zero64 = qweight.quantize(w, bits, scheme, want_fp64=True)
    codes, _, _ = qweight.unpack(qw)
    wb = torch_to_bits(w)
    del w
    got = codes.cpu().numpy()
    del codes
    torch.cuda.empty_cache()
    oc, os_, oz = oracle.port().quantize_matrix(wb, bits, scheme)
    assert got.shape == oc.shape
    bad = np.count_nonzero(got != oc)
    assert bad == 0, f"{bad} codes differ of {got.size}"
    np.testing.assert_array_equal(step64.cpu().numpy().view(np.uint64), os_.view(np.uint64))
    np.testing.assert_array_equal(zero64.cpu().numpy() + 0.0, oz + 0.0)
    assert qw.packed.numel() == -(-n * k * bits // 8)
