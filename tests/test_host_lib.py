"""The B200 build's C++ host library (drop-in hetplan:: re-implementation)
through its C-ABI, against golden values from the reference's own code.
CPU only: these never touch the GPU."""
import ctypes as C

import numpy as np
import pytest

from paper_2403_01136_b200 import capi
from paper_2403_01136_b200.capi import check, lib

D = C.POINTER(C.c_double)


def _csv(stats_csv, bits, scheme, rounding):
    b = (C.c_int * len(bits))(*bits)
    buf = C.create_string_buffer(1 << 20)
    check(lib.hp_host_indicator_csv(stats_csv.encode(), b, len(bits), scheme, rounding, buf,
                                    len(buf)))
    return buf.value.decode()


def test_indicator_tables_bit_identical(planning_golden):
    g = planning_golden
    assert _csv(g["sample_calibration_csv"], [3, 4, 8, 16], 1, 0) == g["omega_sample_sym_nearest"]
    assert _csv(g["sample_calibration_csv"], [2, 3, 4, 8, 16], 0, 1) == g["omega_sample_asym_stoch"]
    assert _csv(g["random_stats_csv"], [3, 4, 8, 16], 1, 0) == g["omega_random_sym_nearest"]


def test_indicator_errors_are_invalid_argument(planning_golden):
    with pytest.raises(capi.InvalidArgument):
        _csv("layer,operator\n", [3, 16], 1, 0)
    with pytest.raises(capi.InvalidArgument):  # 16 missing from the bit set
        _csv(planning_golden["sample_calibration_csv"], [3, 4], 1, 0)
    bad = "layer,operator,d_w,w_min,w_max,x_mean,x_var\n1,qkv,4,-1,1,0,1\n"
    with pytest.raises(capi.InvalidArgument):  # layers not contiguous from 0
        _csv(bad, [4, 16], 1, 0)


def test_scaling_factor_and_g_of_x(planning_golden):
    out = C.c_double()
    for a, b, bit, s, want in planning_golden["scaling_factor"]:
        check(lib.hp_host_scaling_factor(a, b, bit, s, C.byref(out)))
        assert out.value == want
    for m, v, r, want in planning_golden["g_of_x"]:
        check(lib.hp_host_g_of_x(m, v, r, C.byref(out)))
        assert out.value == want
    with pytest.raises(capi.InvalidArgument):
        check(lib.hp_host_scaling_factor(1.0, 0.0, 4, 1, C.byref(out)))
    with pytest.raises(capi.InvalidArgument):
        check(lib.hp_host_scaling_factor(0.0, 1.0, 1, 1, C.byref(out)))


def test_memcost_and_presets(planning_golden):
    for name, f in planning_golden["models"].items():
        if name != "opt-125m":
            got = (C.c_int64 * 9)()
            check(lib.hp_host_preset(name.encode(), got))
            assert list(got) == f
        for bit, want in planning_golden["memcost"][name].items():
            out = (C.c_int64 * 3)()
            check(lib.hp_host_memcost((C.c_int64 * 9)(*f), int(bit), 32, 512, 100, out))
            assert list(out) == want, (name, bit)


def test_schedules(planning_golden):
    for B, eta, xi, sizes, groups, ng in planning_golden["schedules"]:
        s = (C.c_int * B)()
        g = (C.c_int * B)()
        nb, ngo = C.c_int(), C.c_int()
        check(lib.hp_host_make_schedule(B, eta, xi, s, g, C.byref(nb), C.byref(ngo), B))
        assert list(s[:nb.value]) == sizes and list(g[:nb.value]) == groups and ngo.value == ng
    with pytest.raises(capi.InvalidArgument):
        check(lib.hp_host_make_schedule(8, 5, 4, s, g, C.byref(nb), C.byref(ngo), 8))


def test_simulate_bit_identical(planning_golden):
    for case in planning_golden["simulate"]:
        costs = np.array(case["costs"], dtype=np.float64)
        S = costs.shape[0]
        out = (C.c_double * 4)()
        busy = (C.c_double * S)()
        cap = case["events"]
        tl = np.zeros((cap, 6))
        check(lib.hp_host_simulate(costs.ctypes.data_as(D), S, case["B"], case["eta"],
                                   case["xi"], case["n"], out, busy, tl.ctypes.data, cap))
        assert out[0] == case["makespan"]
        assert out[1] == case["bubble"]
        assert out[2] == case["analytic"]
        assert int(out[3]) == case["events"]
        assert list(busy) == case["busy"]
        np.testing.assert_array_equal(tl[:len(case["timeline_head"])],
                                      np.array(case["timeline_head"]))


def test_known_pipesim_answers():
    """SPEC.md:501-502 / SURVEY App. B closed forms."""
    out = (C.c_double * 4)()
    busy = (C.c_double * 2)()
    c = np.array([[1.5, 0.25, 0, 0]])
    check(lib.hp_host_simulate(c.ctypes.data_as(D), 1, 1, 1, 1, 11, out, busy, None, 0))
    assert out[0] == 4.0 and out[2] == 1.75
    c = np.array([[2.0, 0.1, 0, 0], [2.0, 0.1, 0, 0]])
    check(lib.hp_host_simulate(c.ctypes.data_as(D), 2, 4, 1, 4, 1, out, busy, None, 0))
    assert out[0] == 10.0
