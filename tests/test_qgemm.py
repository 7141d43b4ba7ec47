"""K3 (decode, M = xi) / K4 (prefill, M = eta*s) fused dequant-GEMM on tcgen05.

Oracle: y = x . (zero + (code - off) * step)^T in fp64 (the reference's
dequant formula, indicator.cpp:53, on codes from the reference-pinned K1),
computed by oracle/hp_oracle.c. Tolerance (BASELINE.json north_star):
normwise max|y - y_ref| / max|y_ref| <= 1e-2 for bf16 output with fp32
accumulation; we assert the tighter 8e-3.
"""
import numpy as np
import pytest

from tests.util import bf16_bits_to_f64, bits_to_torch, to_bf16_bits, torch_to_bits

pytestmark = pytest.mark.gpu

TOL = 8e-3


def _case(rng, n, k, m, bits, scheme, dev, x_mean=0.05):
    import torch
    from paper_2403_01136_b200 import qweight
    wb = to_bf16_bits(rng.normal(0, 0.02, (n, k)))
    xb = to_bf16_bits(rng.normal(x_mean, 1.0, (m, k)))
    w = bits_to_torch(wb, dev)
    x = bits_to_torch(xb, dev)
    qw, step64, zero64 = qweight.quantize(w, bits, scheme, want_fp64=True)
    codes, _, _ = qweight.unpack(qw)
    return qw, x, xb, codes.cpu().numpy(), step64, zero64, wb


def _oracle(xb, codes, step64, zero64, bits, scheme):
    import oracle
    if bits == 16:
        return oracle.port().qlinear(xb, codes.view(np.uint16), None, None, 16, scheme)
    return oracle.port().qlinear(xb, codes, step64.cpu().numpy(), zero64.cpu().numpy(), bits,
                                 scheme)


def _err(got, ref):
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))


@pytest.mark.parametrize("bits", (3, 4, 8, 16))
@pytest.mark.parametrize("scheme", (0, 1))
@pytest.mark.parametrize("m,phase", [(8, 1), (32, 1), (1, 1), (13, 1), (512, 0), (200, 0)])
def test_qlinear_vs_oracle(cuda, bits, scheme, m, phase):
    if bits == 16 and scheme == 0:
        pytest.skip("16-bit has no scheme")
    from paper_2403_01136_b200 import qweight
    rng = np.random.default_rng(bits * 100 + scheme * 10 + m)
    n, k = 384, 640
    qw, x, xb, codes, s64, z64, _ = _case(rng, n, k, m, bits, scheme, cuda)
    y = qweight.qlinear(qw, x, phase=phase)
    got = bf16_bits_to_f64(torch_to_bits(y))
    ref = _oracle(xb, codes, s64, z64, bits, scheme).astype(np.float64)
    e = _err(got, ref)
    assert e <= TOL, f"normwise err {e}"


@pytest.mark.parametrize("n,k", [(768, 768), (2304, 768), (3072, 768), (768, 3072)])
def test_opt125m_shapes_decode_and_prefill(cuda, n, k):
    """OPT-125M op shapes (qkv/out/fc1/fc2) at xi=8 decode and a 512-token
    prefill micro-batch, against a torch fp32 reference of the dequantized
    weights."""
    import torch
    from paper_2403_01136_b200 import qweight
    rng = np.random.default_rng(n + k)
    for bits in (4, 8):
        for m, phase in ((8, 1), (512, 0)):
            qw, x, xb, codes, s64, z64, _ = _case(rng, n, k, m, bits, 1, cuda)
            off = (1 << (bits - 1)) - 1
            wdq = (torch.from_numpy(codes.astype(np.float64) - off).to(cuda) *
                   s64.repeat_interleave(128, dim=1)[:, :k])
            ref = (x.double() @ wdq.T).float().cpu().numpy()
            got = qweight.qlinear(qw, x, phase=phase).float().cpu().numpy()
            assert _err(got, ref) <= TOL


def test_epilogues_residual_and_relu(cuda):
    import torch
    from paper_2403_01136_b200 import qweight
    rng = np.random.default_rng(11)
    n, k = 512, 768
    for m, phase in ((8, 1), (300, 0)):
        qw, x, xb, codes, s64, z64, _ = _case(rng, n, k, m, 4, 1, cuda)
        res = (torch.randn(m, n, device=cuda)).to(torch.bfloat16)
        base = _oracle(xb, codes, s64, z64, 4, 1).astype(np.float64)
        y_relu = qweight.qlinear(qw, x, phase=phase, relu=True)
        assert _err(y_relu.float().cpu().numpy(), np.maximum(base, 0)) <= TOL
        y_res = qweight.qlinear(qw, x, phase=phase, residual=res)
        want = base + res.float().cpu().numpy()
        assert _err(y_res.float().cpu().numpy(), want) <= TOL


def test_strided_activation_and_output(cuda):
    """x is a column slice of a wider buffer (the V third of a qkv output)."""
    import torch
    from paper_2403_01136_b200 import qweight
    rng = np.random.default_rng(5)
    n, k, m = 256, 512, 32
    qw, _, _, codes, s64, z64, _ = _case(rng, n, k, m, 4, 1, cuda)
    big = (torch.randn(m, 3 * k, device=cuda)).to(torch.bfloat16)
    x = big[:, 2 * k:]
    out = torch.zeros(m, 2 * n, dtype=torch.bfloat16, device=cuda)
    qweight.qlinear(qw, x, phase=1, out=out[:, n:])
    ref = _oracle(torch_to_bits(x.contiguous()), codes, s64, z64, 4, 1)
    assert _err(out[:, n:].float().cpu().numpy(), ref) <= TOL
    assert torch.count_nonzero(out[:, :n]) == 0


@pytest.mark.parametrize("bits", (3, 4, 8, 16))
def test_decode_stream_k_is_deterministic(cuda, bits):
    """Stream-K partials are reduced in segment order: bit-identical reruns.
    Also guards the round-robin ring-depth rule (a parity-aliasing race
    showed up as garbage on some launches, not all)."""
    import torch
    from paper_2403_01136_b200 import qweight
    rng = np.random.default_rng(3)
    qw, x, *_ = _case(rng, 1024, 7168, 32, bits, 1, cuda)
    a = qweight.qlinear(qw, x, phase=1)
    assert torch.isfinite(a.float()).all()
    for _ in range(5):
        assert torch.equal(a, qweight.qlinear(qw, x, phase=1))


@pytest.mark.parametrize("bits", (3, 4, 8, 16))
def test_large_shape_decode(cuda, bits):
    """OPT-30B fc2 shape [7168 x 28672] at xi=32: split-K path end to end,
    checked against torch fp32 on the dequantized weights."""
    import torch
    from paper_2403_01136_b200 import qweight
    n, k, m = 7168, 28672, 32
    w = (torch.randn(n, k, device=cuda) * 0.02).to(torch.bfloat16)
    x = (torch.randn(m, k, device=cuda) + 0.05).to(torch.bfloat16)
    qw = qweight.quantize(w, bits)
    wdq = qweight.dequant(qw).float()
    ref = (x.float() @ wdq.T)
    got = qweight.qlinear(qw, x, phase=1).float()
    e = float((got - ref).abs().max() / ref.abs().max())
    assert e <= TOL


def test_shared_workspace_across_tile_counts(cuda):
    """One split-K workspace serves ops with different tile counts (the
    pipeline shares one per stage): an op with few tiles (large partial
    region start) must not leave data in another op's tile tickets.
    Regression: out-proj [5120 x 5120] (40 tiles) before fc1 [20480 x 5120]
    (160 tiles, > 148 SMs) corrupted fc1's split tiles >= 128."""
    import torch
    from paper_2403_01136_b200 import qweight
    g = torch.Generator(device="cpu").manual_seed(7)
    small = qweight.quantize((torch.randn(5120, 5120, generator=g) * 0.02).to(torch.bfloat16).to(cuda), 4)
    big = qweight.quantize((torch.randn(20480, 5120, generator=g) * 0.02).to(torch.bfloat16).to(cuda), 4)
    x = torch.randn(32, 5120, generator=g).to(torch.bfloat16).to(cuda)
    fresh = qweight.qlinear(big, x, workspace=qweight.Workspace(cuda))
    ws = qweight.Workspace(cuda)
    qweight.qlinear(small, x, workspace=ws)
    chained = qweight.qlinear(big, x, workspace=ws)
    torch.cuda.synchronize()
    assert torch.equal(fresh, chained)


@pytest.mark.parametrize("bits", (3, 16))
def test_prefill_many_token_tiles_ragged(cuda, bits):
    """A long prefill (149 BN=256 token tiles, one more than the persistent
    grid, the last one ragged) matches the oracle: every CTA walks several
    tiles and the partial tile's rows are masked."""
    from paper_2403_01136_b200 import qweight
    rng = np.random.default_rng(4242 + bits)
    n, k, m = 128, 256, 256 * 149 - 77
    qw, x, xb, codes, s64, z64, _ = _case(rng, n, k, m, bits, 1, cuda)
    y = qweight.qlinear(qw, x, phase=0)
    got = bf16_bits_to_f64(torch_to_bits(y))
    ref = _oracle(xb, codes, s64, z64, bits, 1).astype(np.float64)
    assert _err(got, ref) <= TOL


@pytest.mark.parametrize("bits", (4, 16))
def test_prefill_data_parallel_plus_stream_k(cuda, bits, monkeypatch):
    """A wave-quantised prefill op (320 BN=256 tiles = 2.16 waves of 148
    CTAs) runs its first wave as whole tiles and the rest as stream-K
    group ranges when HP_PREFILL_DP_WAVES=1; both that split and the default
    pure stream-K split match the oracle, and each is deterministic."""
    import torch
    from paper_2403_01136_b200 import qweight
    rng = np.random.default_rng(777 + bits)
    n, k, m = 5120, 512, 2048
    qw, x, xb, codes, s64, z64, _ = _case(rng, n, k, m, bits, 1, cuda)
    ref = _oracle(xb, codes, s64, z64, bits, 1).astype(np.float64)
    for waves in (None, "1"):
        if waves is None:
            monkeypatch.delenv("HP_PREFILL_DP_WAVES", raising=False)
        else:
            monkeypatch.setenv("HP_PREFILL_DP_WAVES", waves)
        y = qweight.qlinear(qw, x, phase=0)
        for _ in range(5):  # the pre-fix cross-proxy race showed in ~1 of 6 calls
            assert torch.equal(y, qweight.qlinear(qw, x, phase=0))
        got = bf16_bits_to_f64(torch_to_bits(y))
        assert _err(got, ref) <= TOL, waves
