"""The C-ABI boundary: every function declared in include/hp_capi.h is
exported by libhetplan_b200.so, and without a B200 the compute entry points
fail loudly (HP_ECUDA) instead of falling back to the CPU. CPU only."""
import re
from pathlib import Path

import pytest

from paper_2403_01136_b200 import capi

HEADER = Path(__file__).resolve().parents[1] / "include" / "hp_capi.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    names = re.findall(r"\b(hp_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(capi.lib, n)]
    assert not missing, missing
    assert set(capi.EXPORTED) <= set(names)


def test_abi_version_and_sizes():
    assert capi.lib.hp_abi_version() == 2
    # packed-size contract (memcost.cpp:15-18): ceil(n*k*b/8) on aligned shapes
    for bits in (3, 4, 8, 16):
        assert capi.lib.hp_packed_bytes(5120, 20480, bits) == 5120 * 20480 * bits // 8
    assert capi.lib.hp_packed_bytes(0, 10, 4) == -1
    assert capi.lib.hp_packed_bytes(10, 10, 5) == -1
    assert capi.lib.hp_scale_count(256, 300) == 2 * 3 * 128


@pytest.mark.skipif(capi.device_ok(), reason="a B200 is present")
def test_no_cpu_fallback_without_device():
    import ctypes as C
    st = capi.lib.hp_quant_pack(C.c_void_p(16), 128, 128, 128, 4, 1, 0, C.c_void_p(16),
                                C.c_void_p(16), None, None, None, None)
    assert st == capi.HP_ECUDA
    assert b"no usable sm_100" in capi.lib.hp_last_error()
    w = capi.hp_qweight(128, 128, 4, 1, 16, 16, None)
    st = capi.lib.hp_qlinear(C.byref(w), C.c_void_p(16), 128, 8, C.c_void_p(16), 128, None, 0,
                             0, capi.HP_DECODE, None, 0, None)
    assert st == capi.HP_ECUDA


def test_invalid_arguments_are_einval():
    import ctypes as C
    st = capi.lib.hp_quant_pack(None, 128, 128, 128, 4, 1, 0, None, None, None, None, None, None)
    assert st == capi.HP_EINVAL
    st = capi.lib.hp_quant_pack(C.c_void_p(16), 128, 128, 128, 5, 1, 0, C.c_void_p(16),
                                C.c_void_p(16), None, None, None, None)
    assert st == capi.HP_EINVAL
    st = capi.lib.hp_quant_pack(C.c_void_p(16), 128, 128, 128, 4, 1, capi.HP_STOCHASTIC,
                                C.c_void_p(16), C.c_void_p(16), None, None, None, None)
    assert st == capi.HP_EINVAL and b"round-to-nearest" in capi.lib.hp_last_error()


def test_plan_documents_round_trip_and_validate():
    import ctypes as C
    import json
    plans = Path(__file__).resolve().parent / "golden" / "plans"
    for f in sorted([*plans.glob("*gpu.json"), *plans.glob("*gpu_weak.json")]):
        buf = C.create_string_buffer(1 << 20)
        capi.check(capi.lib.hp_host_plan_check(f.read_bytes(), buf, len(buf)))
        a, b = json.loads(f.read_text()), json.loads(buf.value)
        for k in ("layer_bits", "eta", "xi", "device_order", "objective"):
            assert a[k] == b[k], (f.name, k)
        assert [s["layers"] for s in a["stages"]] == [s["layers"] for s in b["stages"]]
    bad = json.loads((plans / "opt13b_b32_1gpu.json").read_text())
    bad["layer_bits"][0] = 5
    with pytest.raises(capi.InvalidArgument):
        capi.check(capi.lib.hp_host_plan_check(json.dumps(bad).encode(), buf, len(buf)))


def test_plan_format_2_round_trip():
    """Plan JSON v2: serialize writes format_version 2,
    the quant block and device_index = stage index; v2 reloads to the same
    plan; reference-format (v1) documents still load; bad quant rejected."""
    import ctypes as C
    import json
    plans = Path(__file__).resolve().parent / "golden" / "plans"
    for f in sorted([*plans.glob("*gpu.json"), *plans.glob("*gpu_weak.json")]):
        buf = C.create_string_buffer(1 << 20)
        capi.check(capi.lib.hp_host_plan_check(f.read_bytes(), buf, len(buf)))
        v2 = json.loads(buf.value)
        assert v2["format_version"] == 2
        assert v2["quant"] == {"group": 128, "scheme": "symmetric", "rounding": "nearest",
                               "layout": "hp-tile-128x128-v1"}
        assert [s["device_index"] for s in v2["stages"]] == list(range(len(v2["stages"])))
        buf2 = C.create_string_buffer(1 << 20)
        capi.check(capi.lib.hp_host_plan_check(buf.value, buf2, len(buf2)))
        assert json.loads(buf2.value) == v2  # fixed point
    base = json.loads(buf.value)
    for key, val in (("group", 64), ("scheme", "nf4"), ("rounding", "stochastic"), ("layout", "gptq")):
        bad = json.loads(json.dumps(base))
        bad["quant"][key] = val
        with pytest.raises(capi.InvalidArgument):
            capi.check(capi.lib.hp_host_plan_check(json.dumps(bad).encode(), buf2, len(buf2)))
    bad = json.loads(json.dumps(base))
    bad["format_version"] = 3
    with pytest.raises(capi.InvalidArgument):
        capi.check(capi.lib.hp_host_plan_check(json.dumps(bad).encode(), buf2, len(buf2)))


def test_cpp_wrappers_keep_reference_exception_contract(tmp_path):
    """include/hetplan/{quant,qlinear}.hpp rethrow hp_status as the reference's
    exception types: invalid_argument / runtime_error."""
    import subprocess
    root = Path(__file__).resolve().parents[1]
    lib = root / "paper_2403_01136_b200" / "libhetplan_b200.so"
    exe = tmp_path / "wrappers"
    r = subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", f"-I{root / 'include'}",
                        str(root / "tests" / "dropin" / "wrappers_main.cpp"), "-o", str(exe),
                        f"-L{lib.parent}", "-lhetplan_b200", f"-Wl,-rpath,{lib.parent}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0 and "wrappers: ok" in r.stdout, r.stdout + r.stderr
