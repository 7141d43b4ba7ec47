"""Latency model (hetplan::latcost, our Eigen-free re-implementation of
/root/reference/proj/src/latcost.cpp) through the C-ABI, CPU only.

Known answers are the reference SPEC's latcost examples:
exact synthesize-then-fit recovery within 1e-9 absolute, constant samples
-> intercept only (1e-12), duplicate averaging, errors on nonpositive
latency / too few samples / rank-deficient designs, predictions clamped at
zero; plus agreement with numpy's least squares on noisy profiles.
"""
import ctypes as C
import json

import numpy as np
import pytest

from paper_2403_01136_b200 import capi
from paper_2403_01136_b200.capi import lib

HDR = "device,bit,phase,v,s,t,latency_s\n"


def fit(csv: str) -> dict:
    need = C.c_int64()
    buf = C.create_string_buffer(1 << 16)
    capi.check(lib.hp_host_latency_fit(csv.encode(), buf, len(buf), C.byref(need)))
    return json.loads(buf.value.decode())


def status(csv: str) -> int:
    buf = C.create_string_buffer(1 << 16)
    return lib.hp_host_latency_fit(csv.encode(), buf, len(buf), None)


def predict(model: dict, dev, bit, phase, v, s, t=0.0) -> float:
    out = C.c_double()
    capi.check(lib.hp_host_latency_predict(json.dumps(model).encode(), dev.encode(), bit, phase, v, s,
                                           t, C.byref(out)))
    return out.value


def coeffs(model, dev, bit, phase):
    for g in model["groups"]:
        if g["device"] == dev and g["bit"] == bit and g["phase"] == phase:
            return np.array(g["coeffs"])
    raise KeyError


def pre_feat(v, s):
    return np.array([1.0, v, s, v * s, v * s * s])


def dec_feat(v, s, t):
    return np.array([1.0, v, v * (t + s), t + s])


def test_spec_exact_prefill_fit():
    truth = np.array([0.001, 0.002, 0.0001, 5e-5, 1e-8])
    pts = [(v, s) for v in (1, 2, 4, 8) for s in (128, 256, 512)]  # 12 distinct points
    rows = "".join(f"b200,4,prefill,{v},{s},0,{float(pre_feat(v, s) @ truth)!r}\n" for v, s in pts)
    m = fit(HDR + rows)
    got = coeffs(m, "b200", 4, "prefill")
    assert np.abs(got - truth).max() <= 1e-9
    assert m["groups"][0]["residuals"]["n"] == 12
    assert m["format_version"] == 1


def test_spec_constant_samples():
    rows = "".join(f"b200,8,decode,{v},{s},{t},0.5\n" for v in (1, 4, 16) for s in (128, 512)
                   for t in (0, 50))
    c = coeffs(fit(HDR + rows), "b200", 8, "decode")
    assert abs(c[0] - 0.5) <= 1e-12 and np.abs(c[1:]).max() <= 1e-12


def test_decode_fit_matches_numpy_lstsq():
    rng = np.random.default_rng(7)
    truth = np.array([5e-6, 1e-7, 4e-10, 2e-9])
    pts = [(v, s, t) for v in (1, 8, 32) for s in (128, 512) for t in (1, 25, 50, 99)]
    X = np.array([dec_feat(*p) for p in pts])
    y = X @ truth * (1 + 0.05 * rng.standard_normal(len(pts)))
    rows = "".join(f"gpu,3,decode,{v},{s},{t},{float(lat)!r}\n" for (v, s, t), lat in zip(pts, y))
    got = coeffs(fit(HDR + rows), "gpu", 3, "decode")
    ref = np.linalg.lstsq(X, y, rcond=None)[0]
    assert np.abs(got - ref).max() <= 1e-9 * np.abs(ref).max()


def test_duplicates_averaged():
    rows = "d,16,prefill,1,0,0,1.0\nd,16,prefill,1,0,0,3.0\n"
    base = "".join(f"d,16,prefill,{v},{s},0,{1.0 + v + s * 1e-3 + v * s * 1e-4 + v * s * s * 1e-7!r}\n"
                   for v, s in ((2, 128), (4, 256), (8, 512), (2, 512), (8, 128)))
    m = fit(HDR + rows + base)
    assert m["groups"][0]["residuals"]["n"] == 6  # the two (1, 0) rows are one sample


@pytest.mark.parametrize("csv,code", [
    (HDR + "d,4,prefill,1,128,0,-1\n", capi.HP_EINVAL),                 # nonpositive latency
    ("device,bit,phase,v,s,latency_s\nd,4,prefill,1,1,1\n", capi.HP_EINVAL),  # header
    (HDR + "d,4,prefill,1,128\n", capi.HP_EINVAL),                      # column count
    (HDR + "d,4,bogus,1,128,0,1\n", capi.HP_EINVAL),                    # phase
    (HDR + "".join(f"d,4,prefill,{v},128,0,1\n" for v in (1, 2, 3)), None),  # 3 < 5 samples
    (HDR + "".join(f"d,4,prefill,{v},128,0,{v}\n" for v in range(1, 9)), None),  # s constant: rank 3
])
def test_errors(csv, code):
    st = status(csv)
    assert st != capi.HP_OK
    if code is not None:
        assert st == code
    else:
        msg = lib.hp_last_error().decode()
        assert "(d, 4-bit, prefill)" in msg


def test_predict_and_clamp():
    m = {"format_version": 1, "groups": [
        {"device": "b200", "bit": 4, "phase": "prefill", "coeffs": [-1.0, 0, 0, 0, 0]},
        {"device": "b200", "bit": 4, "phase": "decode", "coeffs": [1e-5, 2e-6, 3e-9, 4e-8]}]}
    assert predict(m, "b200", 4, 0, 4, 512) == 0.0  # clamped
    want = float(np.array([1e-5, 2e-6, 3e-9, 4e-8]) @ dec_feat(32, 512, 50))
    assert predict(m, "b200", 4, 1, 32, 512, 50) == pytest.approx(want, rel=1e-15)
    out = C.c_double()
    assert lib.hp_host_latency_predict(json.dumps(m).encode(), b"b200", 8, 1, 1, 1, 1, C.byref(out)) != 0


def test_b200_profile_fixture_refits_to_committed_model():
    """tools/latency_profile.py on a B200 wrote the per-layer profile and its
    fitted model (tests/golden/plans/b200_opt13b.*); refitting the committed
    profile reproduces the committed model, and it predicts every profiled
    decode point within its residual bound."""
    from pathlib import Path
    plans = Path(__file__).parent / "golden" / "plans"
    csv = (plans / "b200_opt13b.profile.csv").read_text()
    committed = json.loads((plans / "b200_opt13b.latency_model.json").read_text())
    refit = fit(csv)
    for a, b in zip(refit["groups"], committed["groups"]):
        assert (a["device"], a["bit"], a["phase"]) == (b["device"], b["bit"], b["phase"])
        assert np.allclose(a["coeffs"], b["coeffs"], rtol=1e-12, atol=1e-18)
    for line in csv.strip().splitlines()[1:]:
        dev, bit, ph, v, s, t, lat = line.split(",")
        if ph == "decode":
            g = next(g for g in committed["groups"] if g["bit"] == int(bit) and g["phase"] == "decode")
            got = predict(committed, dev, int(bit), 1, float(v), float(s), float(t))
            assert abs(got - float(lat)) <= g["residuals"]["max_abs"] * (1 + 1e-9) + 1e-15
