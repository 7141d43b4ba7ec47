"""ORACLE — TEST INFRASTRUCTURE ONLY.

Python access to the two CPU checkers of the adaptive-bitwidth linear path:

* ``ref``  — the reference's own code (/root/reference/proj/src compiled by
  oracle/Makefile into oracle/_ref/libhetplan_ref.so; quantize() reached
  through ref_shim.cpp). Pins the restatement below.
* ``port`` — oracle/hp_oracle.c, the plain-C restatement (libhp_oracle.so),
  used as checker on the GPU box and as the timed CPU baseline.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package. The product library never
links or calls it.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libhetplan_ref.so"
PORT_SO = HERE / "libhp_oracle.so"

_d, _i, _i64, _p = C.c_double, C.c_int, C.c_int64, C.c_void_p
_P = C.POINTER


def _arr(a, ctype):
    return a.ctypes.data_as(_P(ctype))


class _Port:
    def __init__(self):
        if not PORT_SO.exists():
            raise ImportError(f"{PORT_SO} missing: run `make -C oracle`")
        lib = C.CDLL(str(PORT_SO))
        lib.hpo_scaling_factor.restype = _d
        lib.hpo_scaling_factor.argtypes = [_d, _d, _i, _i, _P(_i)]
        lib.hpo_g_of_x.restype = _d
        lib.hpo_g_of_x.argtypes = [_d, _d, _i]
        lib.hpo_layer_indicator.restype = _d
        lib.hpo_layer_indicator.argtypes = [_P(_d), _i, _i, _i, _i]
        lib.hpo_quantize_vec.restype = None
        lib.hpo_quantize_vec.argtypes = [_P(_d), _i64, _i, _i, _P(C.c_int32), _P(_d), _P(_d)]
        lib.hpo_quantize_matrix.restype = None
        lib.hpo_quantize_matrix.argtypes = [_p, _i64, _i64, _i, _i, _p, _p, _p]
        lib.hpo_qlinear.restype = None
        lib.hpo_qlinear.argtypes = [_p, _i64, _i64, _p, _p, _p, _i64, _i, _i, _p, _i]
        lib.hpo_x_stats.restype = None
        lib.hpo_x_stats.argtypes = [_p, _i64, _P(_d), _P(_d)]
        lib.hpo_make_schedule.restype = _i
        lib.hpo_make_schedule.argtypes = [_i, _i, _i, _P(_i), _P(_i), _P(_i)]
        self.lib = lib

    def scaling_factor(self, w_min, w_max, bit, scheme):
        err = _i(0)
        v = self.lib.hpo_scaling_factor(w_min, w_max, bit, scheme, C.byref(err))
        if err.value:
            raise ValueError("scaling_factor: invalid input")
        return v

    def g_of_x(self, mean, var, rounding=0):
        return self.lib.hpo_g_of_x(mean, var, rounding)

    def layer_indicator(self, stats5, bit, scheme=1, rounding=0):
        s = np.ascontiguousarray(stats5, dtype=np.float64).reshape(-1, 5)
        return self.lib.hpo_layer_indicator(_arr(s, _d), s.shape[0], bit, scheme, rounding)

    def quantize_vec(self, w, bit, scheme):
        w = np.ascontiguousarray(w, dtype=np.float64)
        codes = np.zeros(len(w), dtype=np.int32)
        step, zero = _d(), _d()
        self.lib.hpo_quantize_vec(_arr(w, _d), len(w), bit, scheme, _arr(codes, C.c_int32),
                                  C.byref(step), C.byref(zero))
        return codes, step.value, zero.value

    def quantize_matrix(self, w_bits: np.ndarray, bit, scheme):
        """w_bits: uint16 bf16 bit patterns [n_out, k_in]."""
        w_bits = np.ascontiguousarray(w_bits, dtype=np.uint16)
        n, k = w_bits.shape
        G = -(-k // 128)
        codes = np.zeros((n, k), dtype=np.uint8)
        step = np.zeros((n, G))
        zero = np.zeros((n, G))
        self.lib.hpo_quantize_matrix(w_bits.ctypes.data, n, k, bit, scheme, codes.ctypes.data,
                                     step.ctypes.data, zero.ctypes.data)
        return codes, step, zero

    def qlinear(self, x_bits, codes, step, zero, bit, scheme, threads=0):
        x_bits = np.ascontiguousarray(x_bits, dtype=np.uint16)
        m, k = x_bits.shape
        n = codes.shape[0]
        y = np.zeros((m, n), dtype=np.float32)
        codes = np.ascontiguousarray(codes)
        st = np.ascontiguousarray(step, dtype=np.float64) if step is not None else np.zeros(1)
        zr = np.ascontiguousarray(zero, dtype=np.float64) if zero is not None else np.zeros(1)
        self.lib.hpo_qlinear(x_bits.ctypes.data, m, k, codes.ctypes.data, st.ctypes.data,
                             zr.ctypes.data, n, bit, scheme, y.ctypes.data, threads)
        return y

    def x_stats(self, x_bits):
        x_bits = np.ascontiguousarray(x_bits, dtype=np.uint16).ravel()
        mean, var = _d(), _d()
        self.lib.hpo_x_stats(x_bits.ctypes.data, x_bits.size, C.byref(mean), C.byref(var))
        return mean.value, var.value

    def make_schedule(self, B, eta, xi):
        m = -(-B // eta) if eta > 0 else 0
        sizes = (C.c_int * max(m, 1))()
        groups = (C.c_int * max(m, 1))()
        ng = _i()
        r = self.lib.hpo_make_schedule(B, eta, xi, sizes, groups, C.byref(ng))
        if r < 0:
            raise ValueError("make_schedule: invalid")
        return list(sizes[:r]), list(groups[:r]), ng.value


class _Ref:
    """The reference's own compiled code (needs oracle/_ref built here)."""

    def __init__(self):
        if not REF_SO.exists():
            raise ImportError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        lib = C.CDLL(str(REF_SO))
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_quantize.argtypes = [_P(_d), _i64, _i, _i, _i, C.c_uint64, _P(_d)]
        lib.ref_scaling_factor.argtypes = [_d, _d, _i, _i, _P(_d)]
        lib.ref_g_of_x.argtypes = [_d, _d, _i, _P(_d)]
        lib.ref_indicator_csv.argtypes = [C.c_char_p, _P(_i), _i, _i, _i, C.c_char_p, _i64]
        lib.ref_mc_output_variance.argtypes = [_P(_d), _i64, _d, _d, _i, _i, _i, _i64, C.c_uint64, _P(_d)]
        lib.ref_memcost.argtypes = [_P(_i64), _i, _i64, _i64, _i64, _P(_i64)]
        lib.ref_preset.argtypes = [C.c_char_p, _P(_i64)]
        lib.ref_make_schedule.argtypes = [_i, _i, _i, _P(_i), _P(_i), _P(_i), _P(_i), _i]
        lib.ref_simulate.argtypes = [_P(_d), _i, _i, _i, _i, _i, _P(_d), _P(_d), _p, _i64]
        lib.ref_validate_plan.argtypes = [_P(_i), _i, _P(_i), _i, _P(_i), _i, _i, _i, _P(_d),
                                          _i, _i, _i, _P(_i), _i]
        lib.ref_best_plan.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, _d, _i, _i, _d,
                                      C.c_char_p, _i64]
        self.lib = lib

    def _chk(self, rc):
        if rc != 0:
            msg = self.lib.ref_last_error().decode()
            if rc == 2:
                raise ValueError(msg)
            raise RuntimeError(msg)

    def quantize(self, w, bit, scheme, rounding=0, seed=0):
        w = np.ascontiguousarray(w, dtype=np.float64)
        out = np.zeros_like(w)
        self._chk(self.lib.ref_quantize(_arr(w, _d), len(w), bit, scheme, rounding, seed,
                                        _arr(out, _d)))
        return out

    def quantize_codes(self, w, bit, scheme):
        """Reference quantize() -> (signed codes, step, zero); codes recovered
        exactly as lround((out - zero) / step)."""
        w = np.ascontiguousarray(w, dtype=np.float64)
        out = self.quantize(w, bit, scheme)
        step = self.scaling_factor(float(w.min()), float(w.max()), bit, scheme)
        zero = float(w.min()) if scheme == 0 else 0.0
        if step == 0.0:
            return np.zeros(len(w), dtype=np.int32), step, zero
        codes = np.rint((out - zero) / step).astype(np.int32)
        return codes, step, zero

    def scaling_factor(self, w_min, w_max, bit, scheme):
        v = _d()
        self._chk(self.lib.ref_scaling_factor(w_min, w_max, bit, scheme, C.byref(v)))
        return v.value

    def g_of_x(self, mean, var, rounding=0):
        v = _d()
        self._chk(self.lib.ref_g_of_x(mean, var, rounding, C.byref(v)))
        return v.value

    def indicator_csv(self, stats_csv: str, bits, scheme=1, rounding=0) -> str:
        b = (C.c_int * len(bits))(*bits)
        buf = C.create_string_buffer(1 << 20)
        self._chk(self.lib.ref_indicator_csv(stats_csv.encode(), b, len(bits), scheme, rounding,
                                             buf, len(buf)))
        return buf.value.decode()

    def mc_output_variance(self, w, mean, var, bit, scheme, rounding, samples, seed):
        w = np.ascontiguousarray(w, dtype=np.float64)
        out = (C.c_double * 4)()
        self._chk(self.lib.ref_mc_output_variance(_arr(w, _d), len(w), mean, var, bit, scheme,
                                                  rounding, samples, seed, out))
        return list(out)

    def preset(self, name):
        f = (C.c_int64 * 9)()
        self._chk(self.lib.ref_preset(name.encode(), f))
        return list(f)

    def memcost(self, model9, bit, v, s, n):
        f = (C.c_int64 * 9)(*model9)
        out = (C.c_int64 * 3)()
        self._chk(self.lib.ref_memcost(f, bit, v, s, n, out))
        return list(out)

    def make_schedule(self, B, eta, xi):
        cap = max(B, 1)
        sizes = (C.c_int * cap)()
        groups = (C.c_int * cap)()
        nb, ng = _i(), _i()
        self._chk(self.lib.ref_make_schedule(B, eta, xi, sizes, groups, C.byref(nb),
                                             C.byref(ng), cap))
        return list(sizes[:nb.value]), list(groups[:nb.value]), ng.value

    def simulate(self, costs, B, eta, xi, n, timeline=False):
        costs = np.ascontiguousarray(costs, dtype=np.float64).reshape(-1, 4)
        S = costs.shape[0]
        out = (C.c_double * 4)()
        busy = (C.c_double * S)()
        cap = 0
        tl = None
        if timeline:
            sched = self.make_schedule(B, eta, xi)
            cap = (len(sched[0]) + sched[2] * max(n - 1, 0)) * S
            tl = np.zeros((cap, 6))
        self._chk(self.lib.ref_simulate(_arr(costs, _d), S, B, eta, xi, n, out, busy,
                                        tl.ctypes.data if tl is not None else None, cap))
        res = {"makespan": out[0], "bubble": out[1], "analytic": out[2],
               "events": int(out[3]), "busy": list(busy)}
        if timeline:
            res["timeline"] = tl[: int(out[3])]
        return res

    def best_plan(self, config_json: str, omega_csv: str, lat_json: str, theta: float,
                  group: int = 1, heuristic: bool = False, time_limit_s: float = 60.0) -> str:
        buf = C.create_string_buffer(1 << 20)
        self._chk(self.lib.ref_best_plan(config_json.encode(), omega_csv.encode(),
                                         lat_json.encode(), theta, group, int(heuristic),
                                         time_limit_s, buf, len(buf)))
        return buf.value.decode()


_port = None
_ref = None


def port() -> _Port:
    global _port
    if _port is None:
        _port = _Port()
    return _port


def ref() -> _Ref:
    global _ref
    if _ref is None:
        _ref = _Ref()
    return _ref


def ref_available() -> bool:
    return REF_SO.exists()
