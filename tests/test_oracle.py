"""The oracle itself, pinned before it is trusted (CPU only).

* oracle port (oracle/hp_oracle.c) vs the golden vectors produced by the
  reference's own compiled code (tests/golden/make_golden.py);
* when oracle/_ref is built here, the reference vs the same golden vectors
  and the SPEC / SURVEY known answers.
"""
import numpy as np
import pytest

import oracle


@pytest.fixture(scope="module")
def port():
    return oracle.port()


def test_port_quantize_vectors_match_golden(port, quant_golden):
    names = {k.split("/")[1] for k in quant_golden.files if k.startswith("vec/")}
    assert len(names) >= 10
    for name in sorted(names):
        w = quant_golden[f"vec/{name}/w"]
        for bits in (3, 4, 8):
            for scheme in (0, 1):
                key = f"vec/{name}/b{bits}s{scheme}"
                codes, step, zero = port.quantize_vec(w, bits, scheme)
                gs, gz = quant_golden[key + "/stepzero"]
                assert step == gs and zero == gz, key
                np.testing.assert_array_equal(codes, quant_golden[key + "/codes"], err_msg=key)


def test_port_quantize_matrix_matches_golden(port, quant_golden):
    for tag in ("aligned", "ragged"):
        wb = quant_golden[f"mat/{tag}/w_bits"]
        for bits in (3, 4, 8):
            for scheme in (0, 1):
                key = f"mat/{tag}/b{bits}s{scheme}"
                c, s, z = port.quantize_matrix(wb, bits, scheme)
                np.testing.assert_array_equal(c, quant_golden[key + "/codes"])
                np.testing.assert_array_equal(s, quant_golden[key + "/step"])
                np.testing.assert_array_equal(z, quant_golden[key + "/zero"])


def test_appendix_c_known_answers(port):
    """SURVEY App. C rows (reference quantize(), nearest, half-up ties)."""
    row1 = [-3, -2.5, -1.5, -0.5, 0.5, 1.5, 2.5, 3]
    row2 = [-0.5, -0.25, 0, 0.125, 0.3125, 0.4375, 0.5, 1.0]
    c, s, z = port.quantize_vec(row1, 3, 1)
    assert list(c) == [-3, -2, -1, 0, 1, 2, 3, 3] and s == 1.0
    assert list(port.quantize_vec(row2, 4, 0)[0]) == [0, 3, 5, 6, 8, 9, 10, 15]
    assert list(port.quantize_vec(row2, 8, 0)[0]) == [0, 43, 85, 106, 138, 159, 170, 255]
    assert list(port.quantize_vec(row2, 8, 1)[0]) == [-63, -32, 0, 16, 40, 56, 64, 127]


def test_spec_indicator_known_answers(port):
    # SPEC.md:280-298
    assert port.scaling_factor(0.0, 2.55, 8, 0) == 0.0099999999999999985
    assert port.scaling_factor(-7.0, 7.0, 4, 1) == 1.0
    assert port.g_of_x(2.0, 1.0, 1) == 5.0 / 6.0
    assert port.layer_indicator([2, -1, 1, 0, 1], 4, 1, 0) == 1.0 / 98.0
    assert port.layer_indicator([2, -1, 1, 0, 1], 16, 1, 0) == 0.0


def test_port_indicator_matches_golden_table(port, planning_golden):
    rows = planning_golden["sample_calibration_csv"].strip().splitlines()[1:]
    stats = {}
    for r in rows:
        f = r.split(",")
        stats.setdefault(int(f[0]), []).append([float(f[2])] + [float(v) for v in f[3:]])
    table = planning_golden["omega_sample_sym_nearest"].strip().splitlines()[1:]
    for line in table:
        f = line.split(",")
        layer = int(f[0])
        for bit, want in zip((3, 4, 8, 16), f[1:]):
            assert port.layer_indicator(stats[layer], bit, 1, 0) == float(want)


def test_port_schedules_match_golden(port, planning_golden):
    for B, eta, xi, sizes, groups, ng in planning_golden["schedules"]:
        assert port.make_schedule(B, eta, xi) == (sizes, groups, ng)


def test_port_qlinear_formula():
    """Tiny hand-computed case of the dequant GEMV (indicator.cpp:53)."""
    from tests.util import to_bf16_bits
    p = oracle.port()
    x = to_bf16_bits(np.array([[1.0, 2.0, 0.5, -1.0]]))
    codes = np.array([[7, 8, 9, 0]], dtype=np.uint8)  # sym 4-bit, off 7
    step = np.array([[0.5]])
    zero = np.array([[0.0]])
    y = p.qlinear(x, codes, step, zero, 4, 1)
    # w = (0, 0.5, 1.0, -3.5) -> 0 + 1 + 0.5 + 3.5
    assert y[0, 0] == 5.0


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built here")
def test_reference_build_reproduces_golden(quant_golden, planning_golden):
    ref = oracle.ref()
    for name in ("appc_row2", "ties_128", "outliers_128"):
        w = quant_golden[f"vec/{name}/w"]
        for bits in (3, 4, 8):
            for scheme in (0, 1):
                c, s, z = ref.quantize_codes(w, bits, scheme)
                np.testing.assert_array_equal(c, quant_golden[f"vec/{name}/b{bits}s{scheme}/codes"])
    assert ref.indicator_csv(planning_golden["sample_calibration_csv"], [3, 4, 8, 16]) == \
        planning_golden["omega_sample_sym_nearest"]
    # SURVEY §8c known answers
    assert ref.memcost(ref.preset("opt-30b"), 16, 32, 512, 100)[0] == 1470787584
    assert ref.memcost(ref.preset("opt-13b"), 4, 32, 512, 100)[1] == 157347840
    assert ref.memcost(ref.preset("opt-13b"), 16, 32, 512, 100)[1] == 629207040
    assert ref.memcost([48, 7168, 28672, 56, 50272, 2050, 7168, 7168, 0], 16, 32, 512, 100)[2] == 561512448
