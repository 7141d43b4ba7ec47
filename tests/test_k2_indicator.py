"""K2 indicator statistics on the GPU -> omega table.

w_min/w_max are exact; x_mean/x_var (population, fp64) within 1e-9 relative
of the oracle's two-pass fp64; omega from GPU stats within 1e-6 of the
reference formula (indicator.cpp:99-127) evaluated on oracle stats, and
bit-identical to it when the stats are identical.
"""
import ctypes as C

import numpy as np
import pytest

from tests.util import bf16_bits_to_f64, bits_to_torch, to_bf16_bits

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,k,t", [(768, 768, 2048), (300, 200, 7), (3072, 768, 512),
                                   (1, 1, 1)])
def test_stats_vs_oracle(cuda, n, k, t):
    import oracle
    from paper_2403_01136_b200 import qweight
    rng = np.random.default_rng(n * 7 + k + t)
    wb = to_bf16_bits(rng.normal(0, 0.02, (n, k)))
    xb = to_bf16_bits(rng.normal(0.05, 1.25, (t, k)))
    s = qweight.indicator_stats(bits_to_torch(wb, cuda), bits_to_torch(xb, cuda)).cpu().numpy()
    wf = bf16_bits_to_f64(wb)
    assert s[0] == n * k
    assert s[1] == wf.min() and s[2] == wf.max()
    mean, var = oracle.port().x_stats(xb)
    assert abs(s[3] - mean) <= 1e-9 * max(abs(mean), 1e-12) + 1e-15
    assert abs(s[4] - var) <= 1e-9 * max(abs(var), 1e-300)


def test_omega_from_gpu_stats(cuda):
    import oracle
    from paper_2403_01136_b200 import capi, qweight
    rng = np.random.default_rng(2403)
    h1, h2, T = 768, 3072, 256
    shapes = [(3 * h1, h1), (h1, h1), (h2, h1), (h1, h2)]
    sigmas = [1.0, 1.25, 1.5, 1.75]
    stats = []
    for layer in range(3):
        for (n, k), sg in zip(shapes, sigmas):
            wb = to_bf16_bits(rng.normal(0, 0.02 * (1 + layer), (n, k)))
            xb = to_bf16_bits(rng.normal(0.05, np.sqrt(sg), (T, k)))
            s = qweight.indicator_stats(bits_to_torch(wb, cuda), bits_to_torch(xb, cuda))
            stats.append(s.cpu().numpy())
    stats = np.array(stats)
    bits = [3, 4, 8, 16]
    om = np.zeros(3 * 4)
    b = (C.c_int * 4)(*bits)
    capi.check(capi.lib.hp_host_omega_from_stats(
        stats.ctypes.data_as(C.POINTER(C.c_double)), 3, 4, b, 4, 1, 0,
        om.ctypes.data_as(C.POINTER(C.c_double))))
    om = om.reshape(3, 4)
    port = oracle.port()
    for layer in range(3):
        for j, bit in enumerate(bits):
            want = port.layer_indicator(stats[4 * layer:4 * layer + 4], bit)
            assert om[layer, j] == want  # same stats -> bit-identical omega
    assert np.all(om[:, 0] >= om[:, 1]) and np.all(om[:, 1] >= om[:, 2])
    assert np.all(om[:, 3] == 0)


@pytest.mark.parametrize("bits", [3, 4, 8, 16])
@pytest.mark.parametrize("n,k,ld", [(768, 768, 768), (300, 200, 200), (1, 1, 1), (257, 1000, 1003),
                                    (2048, 5120, 5120)])
def test_k1_fused_weight_stats(cuda, bits, n, k, ld):
    """hp_quant_pack_stats: K1's pass yields K2's exact w_min / w_max / d_w
     with the packed output unchanged; hp_indicator_stats
    with w = NULL then adds the calibration part without re-reading W."""
    import torch
    from paper_2403_01136_b200 import capi, qweight
    rng = np.random.default_rng(n + 3 * k + bits)
    wfull = to_bf16_bits(rng.normal(0, 0.02, (n, ld)))
    wfull[rng.random((n, ld)) < 1e-3] = to_bf16_bits(np.array([-0.9, 0.7]))[rng.integers(0, 2)]
    wt = bits_to_torch(wfull, cuda)[:, :k]  # ld != k: the unaligned / strided path
    xb = to_bf16_bits(rng.normal(0.05, 1.25, (33, k)))
    x = bits_to_torch(xb, cuda)
    st = torch.full((5,), -7.0, dtype=torch.float64, device=cuda)
    q1 = qweight.quantize(wt, bits, capi.HP_ASYMMETRIC, stats=st)
    s_fused = st.clone().cpu().numpy()
    q2 = qweight.quantize(wt, bits, capi.HP_ASYMMETRIC)
    assert torch.equal(q1.packed, q2.packed)
    if bits != 16:
        assert torch.equal(q1.scale, q2.scale) and torch.equal(q1.zero, q2.zero)
    wf = bf16_bits_to_f64(wfull[:, :k])
    assert s_fused[0] == n * k and s_fused[1] == wf.min() and s_fused[2] == wf.max()
    assert s_fused[3] == -7.0 and s_fused[4] == -7.0  # calibration part untouched
    qweight.indicator_stats(None, x, out=st)
    ref = qweight.indicator_stats(wt, x).cpu().numpy()
    got = st.cpu().numpy()
    assert np.array_equal(got[:3], ref[:3])
    np.testing.assert_allclose(got[3:], ref[3:], rtol=1e-12, atol=1e-15)
