"""K1 quantize+pack on the GPU vs the reference quantizer (bit-exact).

Golden codes/steps/zeros come from the reference's own quantize()
(/root/reference/proj/src/indicator.cpp:19-56) via tests/golden/make_golden.py;
larger shapes are checked against the oracle port (oracle/hp_oracle.c),
itself pinned to the same golden file in test_oracle.py.
"""
import numpy as np
import pytest

from tests.util import bf16_bits_to_f64, bits_to_torch, to_bf16_bits, torch_to_bits

pytestmark = pytest.mark.gpu

BITS = (3, 4, 8)
SCHEMES = (0, 1)


def _quant(w_bits, bits, scheme, dev):
    from paper_2403_01136_b200 import qweight
    w = bits_to_torch(w_bits, dev)
    qw, step64, zero64 = qweight.quantize(w, bits, scheme, want_fp64=True)
    codes, scale, zero = qweight.unpack(qw)
    return qw, codes.cpu().numpy(), step64.cpu().numpy(), zero64.cpu().numpy(), scale, zero


@pytest.mark.parametrize("tag", ["aligned", "ragged"])
@pytest.mark.parametrize("bits", BITS)
@pytest.mark.parametrize("scheme", SCHEMES)
def test_matrix_matches_reference_golden(cuda, quant_golden, tag, bits, scheme):
    wb = quant_golden[f"mat/{tag}/w_bits"]
    key = f"mat/{tag}/b{bits}s{scheme}"
    qw, codes, step64, zero64, scale, zero = _quant(wb, bits, scheme, cuda)
    np.testing.assert_array_equal(codes, quant_golden[key + "/codes"])
    # fp64 step and grid origin: bit-exact (compare as integers)
    np.testing.assert_array_equal(step64.view(np.uint64),
                                  quant_golden[key + "/step"].view(np.uint64))
    np.testing.assert_array_equal(zero64 + 0.0, quant_golden[key + "/zero"] + 0.0)
    # stored fp32 scale/zero are the fp64 values rounded once
    np.testing.assert_array_equal(scale.cpu().numpy(),
                                  quant_golden[key + "/step"].astype(np.float32))
    if scheme == 0:
        np.testing.assert_array_equal(zero.cpu().numpy(),
                                      quant_golden[key + "/zero"].astype(np.float32))


@pytest.mark.parametrize("name", ["appc_row1", "appc_row2", "normal_5", "normal_127",
                                  "normal_128", "outliers_128", "ties_128", "flat_pos",
                                  "flat_zero", "single", "two", "spec_asym_255"])
@pytest.mark.parametrize("bits", BITS)
@pytest.mark.parametrize("scheme", SCHEMES)
def test_vectors_match_reference_golden(cuda, quant_golden, name, bits, scheme):
    w = quant_golden[f"vec/{name}/w"]
    key = f"vec/{name}/b{bits}s{scheme}"
    wb = to_bf16_bits(w)[None, :]
    _, codes, step64, zero64, _, _ = _quant(wb, bits, scheme, cuda)
    off = (1 << (bits - 1)) - 1 if scheme == 1 else 0
    want = quant_golden[key + "/codes"].astype(np.int64) + off
    step, zero = quant_golden[key + "/stepzero"]
    if step == 0.0:  # flat group: the build defines signed code 0
        want = np.full_like(want, off)
    np.testing.assert_array_equal(codes[0].astype(np.int64), want)
    assert step64[0, 0] == step
    assert zero64[0, 0] == zero
    # dequantized value through the reference formula equals the reference's output
    deq = zero + (codes[0].astype(np.float64) - off) * step
    np.testing.assert_array_equal(deq, quant_golden[key + "/out"])


@pytest.mark.parametrize("shape", [(1024, 768), (768, 3072), (384, 1000), (1, 129)])
@pytest.mark.parametrize("bits", BITS)
def test_large_random_vs_oracle_port(cuda, shape, bits):
    import oracle
    rng = np.random.default_rng(hash((shape, bits)) % 2**32)
    w = rng.normal(0, 0.02, shape)
    w[rng.random(shape) < 1e-3] *= 8
    wb = to_bf16_bits(w)
    for scheme in SCHEMES:
        _, codes, step64, zero64, _, _ = _quant(wb, bits, scheme, cuda)
        oc, os_, oz = oracle.port().quantize_matrix(wb, bits, scheme)
        np.testing.assert_array_equal(codes, oc)
        np.testing.assert_array_equal(step64, os_)
        np.testing.assert_array_equal(zero64, oz)


@pytest.mark.parametrize("bits", (3, 4, 8, 16))
def test_packed_size_contract_and_roundtrip(cuda, bits):
    """Packed buffer = ceil(n*k*b/8) (memcost.cpp:15-18); 16-bit is identity."""
    import torch
    from paper_2403_01136_b200 import qweight
    n, k = 768, 3072
    w = (torch.randn(n, k, device=cuda) * 0.02).to(torch.bfloat16)
    qw = qweight.quantize(w, bits)
    assert qw.packed.numel() == -(-n * k * bits // 8)
    codes, _, _ = qweight.unpack(qw)
    if bits == 16:
        assert torch.equal(codes.view(torch.bfloat16), w)
        assert torch.equal(qweight.dequant(qw), w)
    else:
        assert int(codes.max()) < (1 << bits)


def test_dequant_matches_formula(cuda):
    """hp_dequant == bf16(zero + (code-off)*step) within bf16 rounding of the
    scale (3/4-bit use bf16 scale/zero in the MMA operand)."""
    import torch
    from paper_2403_01136_b200 import qweight
    rng = np.random.default_rng(7)
    wb = to_bf16_bits(rng.normal(0, 0.02, (256, 512)))
    for bits in BITS:
        for scheme in SCHEMES:
            qw, codes, step64, zero64, _, _ = _quant(wb, bits, scheme, cuda)
            off = (1 << (bits - 1)) - 1 if scheme == 1 else 0
            ref = zero64.repeat(128, axis=1) + (codes.astype(np.float64) - off) * step64.repeat(128, axis=1)
            got = bf16_bits_to_f64(torch_to_bits(qweight.dequant(qw)))
            err = np.abs(got - ref).max() / np.abs(ref).max()
            assert err < 2 ** -7, (bits, scheme, err)


def test_rejects_stochastic_and_bad_bits(cuda):
    import torch
    from paper_2403_01136_b200 import capi, qweight
    w = torch.zeros(128, 128, dtype=torch.bfloat16, device=cuda)
    with pytest.raises(capi.InvalidArgument):
        qweight.quantize(w, 4, rounding=capi.HP_STOCHASTIC)
    with pytest.raises(capi.InvalidArgument):
        qweight.quantize(w, 5)
