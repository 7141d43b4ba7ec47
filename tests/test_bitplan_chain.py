"""Bit-assignment parity from the build's OWN indicator (VERDICT
r1 item "+2"): GPU K2 statistics -> omega (host indicator,
indicator.cpp:99-127) -> the reference planner (optimizer_planner.cpp:79-170,
the reference's own compiled code in oracle/_ref) -> the SAME layer_bits,
stages, eta and xi as the committed OPT-125M plan fixture, which the
planner proves optimal (machine-independent).

Inputs: the runtime's synthetic OPT-125M weights and calibration
activations (oracle/synth.py bits: weights seed (1, layer, op), calibration
seed (2, layer, op), T = 256 tokens, x ~ N(0.05, sigma_o^2) with
sigma_o^2 = 1.0/1.25/1.5/1.75 for qkv/out/fc1/fc2), exactly what
tests/golden/make_plans.py reduced with the CPU oracle to build the fixture.
"""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

from tests.util import bits_to_torch

pytestmark = pytest.mark.gpu

PLANS = Path(__file__).resolve().parent / "golden" / "plans"
H1, H2, L, T = 768, 3072, 12, 256
SHAPES = [(3 * H1, H1), (H1, H1), (H2, H1), (H1, H2)]
SIG2 = [1.0, 1.25, 1.5, 1.75]
NAMES = ["qkv", "out", "fc1", "fc2"]


def _gpu_stats(dev):
    from oracle import synth
    from paper_2403_01136_b200 import qweight
    out = []
    for i in range(L):
        for o, ((n, k), s2) in enumerate(zip(SHAPES, SIG2)):
            w = bits_to_torch(synth.synth_bits(n * k, synth.seed_for(1, i, o), 0.0, 0.02), dev)
            x = bits_to_torch(synth.synth_bits(T * k, synth.seed_for(2, i, o), 0.05,
                                               float(np.sqrt(s2))), dev)
            out.append(qweight.indicator_stats(w.view(n, k), x.view(T, k)).cpu().numpy())
    return np.array(out)


def test_k2_stats_omega_and_plan_match_fixture(cuda):
    import oracle
    from paper_2403_01136_b200 import capi
    st = _gpu_stats(cuda)
    # 1. K2 stats vs the fixture's calibration CSV (oracle-reduced)
    rows = (PLANS / "opt-125m_calibration_stats.csv").read_text().strip().splitlines()[1:]
    want = np.array([[float(v) for v in r.split(",")[2:]] for r in rows])
    assert want.shape == st.shape
    np.testing.assert_array_equal(st[:, :3], want[:, :3])          # d_w, w_min, w_max exact
    np.testing.assert_allclose(st[:, 3:], want[:, 3:], rtol=1e-9, atol=1e-15)
    # 2. omega: host library on the GPU stats vs the fixture omega (reference
    #    build on the oracle stats)
    bits = [3, 4, 8, 16]
    om = np.zeros(L * 4)
    capi.check(capi.lib.hp_host_omega_from_stats(
        np.ascontiguousarray(st).ctypes.data_as(C.POINTER(C.c_double)), L, 4,
        (C.c_int * 4)(*bits), 4, capi.HP_SYMMETRIC, capi.HP_NEAREST,
        om.ctypes.data_as(C.POINTER(C.c_double))))
    om = om.reshape(L, 4)
    fx = np.array([[float(v) for v in r.split(",")[1:]]
                   for r in (PLANS / "opt125m_b8_1gpu.omega.csv").read_text().strip().splitlines()[1:]])
    np.testing.assert_allclose(om, fx, rtol=1e-9, atol=0)
    # same stats -> bit-identical omega (host library vs the C restatement)
    port = oracle.port()
    for i in range(L):
        for j, b in enumerate(bits):
            assert om[i, j] == port.layer_indicator(st[4 * i:4 * i + 4], b)
    # 3. the reference planner on the GPU-derived omega -> the fixture's plan
    if not oracle.ref_available():
        pytest.skip("oracle/_ref (the reference planner) not built")
    omega_csv = "layer,bit_3,bit_4,bit_8,bit_16\n" + "".join(
        f"{i}," + ",".join(repr(float(v)) for v in om[i]) + "\n" for i in range(L))
    cfg = (PLANS / "opt125m_b8_1gpu.config.json").read_text()
    lat = (PLANS / "opt125m_b8_1gpu.latency.json").read_text()
    plan = json.loads(oracle.ref().best_plan(cfg, omega_csv, lat, 0.001, group=1,
                                             heuristic=False, time_limit_s=60.0))
    ref = json.loads((PLANS / "opt125m_b8_1gpu.json").read_text())
    assert plan["optimal"] and ref["optimal"]
    assert plan["layer_bits"] == ref["layer_bits"]
    assert [s["layers"] for s in plan["stages"]] == [s["layers"] for s in ref["stages"]]
    assert (plan["eta"], plan["xi"]) == (ref["eta"], ref["xi"])
    assert plan["device_order"] == ref["device_order"]
