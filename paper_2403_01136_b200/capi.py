"""ctypes binding of the C-ABI (include/hp_capi.h).

This is the only way Python reaches the product: every GPU entry point is a
call into libhetplan_b200.so. If the library is missing, importing this
module raises — there is no Python or CPU fallback for the path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("HP_LIB_PATH", _PKG / "libhetplan_b200.so"))

HP_OK, HP_EINTERNAL, HP_EINVAL, HP_EINFEASIBLE, HP_ETIMEOUT, HP_ECUDA, HP_ENCCL = 0, 1, 2, 3, 4, 5, 6
HP_ASYMMETRIC, HP_SYMMETRIC = 0, 1
HP_NEAREST, HP_STOCHASTIC = 0, 1
HP_PREFILL, HP_DECODE = 0, 1
HP_EPI_NONE, HP_EPI_RELU = 0, 1


class HPError(RuntimeError):
    """Raised for any non-zero hp_status; `.status` holds the code."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"hp_status {status}: {msg}")
        self.status = status


class InvalidArgument(HPError, ValueError):
    """HP_EINVAL — the reference's std::invalid_argument."""


class Infeasible(HPError):
    """HP_EINFEASIBLE — the reference's hetplan::infeasible_error."""


class hp_qweight(C.Structure):
    _fields_ = [
        ("n_out", C.c_int64),
        ("k_in", C.c_int64),
        ("bits", C.c_int32),
        ("scheme", C.c_int32),
        ("packed", C.c_void_p),
        ("scale", C.c_void_p),
        ("zero", C.c_void_p),
    ]


class hp_pipeline_options(C.Structure):
    _fields_ = [
        ("scheme", C.c_int32),
        ("use_graphs", C.c_int32),
        ("instrument", C.c_int32),
        ("sm_budget", C.c_int32),
        ("seed", C.c_uint64),
        ("weight_std", C.c_double),
        ("timeout_s", C.c_double),
    ]


class hp_tensor_src(C.Structure):
    _fields_ = [("host", C.c_void_p), ("path", C.c_char_p), ("offset", C.c_int64)]


class hp_weight_set(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int32),
        ("linear", C.POINTER(hp_tensor_src)),
        ("norm", C.POINTER(hp_tensor_src)),
        ("embed", hp_tensor_src),
        ("pos", hp_tensor_src),
        ("final_norm", hp_tensor_src * 2),
        ("bin_bytes", C.c_int64),
    ]


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the product has no fallback path)")
    lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    v, i64, i32, d, p = C.c_void_p, C.c_int64, C.c_int, C.c_double, C.c_char_p
    P = C.POINTER
    sig = {
        "hp_last_error": (p, []),
        "hp_abi_version": (i32, []),
        "hp_device_ok": (i32, []),
        "hp_packed_bytes": (i64, [i64, i64, i32]),
        "hp_scale_count": (i64, [i64, i64]),
        "hp_quant_pack": (i32, [v, i64, i64, i64, i32, i32, i32, v, v, v, v, v, v]),
        "hp_quant_pack_stats": (i32, [v, i64, i64, i64, i32, i32, i32, v, v, v, v, v, v, v]),
        "hp_quant_unpack": (i32, [P(hp_qweight), v, v, v, v]),
        "hp_dequant": (i32, [P(hp_qweight), v, v]),
        "hp_indicator_stats": (i32, [v, i64, i64, i64, v, i64, i64, v, v]),
        "hp_qlinear_workspace_bytes": (C.c_size_t, [P(hp_qweight), i64, i32]),
        "hp_qlinear": (i32, [P(hp_qweight), v, i64, i64, v, i64, v, i64, i32, i32, v, C.c_size_t, v]),
        "hp_host_scaling_factor": (i32, [d, d, i32, i32, P(d)]),
        "hp_host_g_of_x": (i32, [d, d, i32, P(d)]),
        "hp_host_indicator_csv": (i32, [p, P(i32), i32, i32, i32, C.c_char_p, i64]),
        "hp_host_omega_from_stats": (i32, [P(d), i32, i32, P(i32), i32, i32, i32, P(d)]),
        "hp_host_mc_output_variance": (i32, [P(d), i64, d, d, i32, i32, i32, i64, C.c_uint64, P(d)]),
        "hp_host_memcost": (i32, [P(i64), i32, i64, i64, i64, P(i64)]),
        "hp_host_preset": (i32, [p, P(i64)]),
        "hp_host_make_schedule": (i32, [i32, i32, i32, P(i32), P(i32), P(i32), P(i32), i32]),
        "hp_host_simulate": (i32, [P(d), i32, i32, i32, i32, i32, P(d), P(d), v, i64]),
        "hp_host_plan_check": (i32, [p, C.c_char_p, i64]),
        "hp_host_unit_order": (i32, [p, p, i32, P(i32), i32, P(i32)]),
        "hp_host_latency_fit": (i32, [p, p, i64, P(i64)]),
        "hp_host_latency_predict": (i32, [p, p, i32, i32, C.c_double, C.c_double, C.c_double, P(C.c_double)]),
    }
    sig.update({
        "hp_set_sm_budget": (None, [i32]),
        "hp_set_pdl": (None, [i32]),
        "hp_nccl_unique_id": (i32, [v]),
        "hp_pipeline_create": (i32, [p, p, i32, i32, v, P(hp_pipeline_options), P(hp_weight_set), P(v)]),
        "hp_pipeline_run": (i32, [v, v, v, P(d)]),
        "hp_pipeline_final_hidden": (i32, [v, v]),
        "hp_pipeline_load_stats": (i32, [v, P(d)]),
        "hp_pipeline_stage_costs": (i32, [v, P(d)]),
        "hp_pipeline_kernel_stats": (i32, [v, i32, P(d)]),
        "hp_pipeline_layer_costs": (i32, [v, i32, P(d), i64, P(i64)]),
        "hp_pipeline_info": (i32, [v, P(i64)]),
        "hp_pipeline_destroy": (None, [v]),
        "hp_mbm_create": (i32, [i32, i32, i32, i32, P(v)]),
        "hp_mbm_prefill_done": (i32, [v, i32, P(i32)]),
        "hp_mbm_decode_done": (i32, [v, i32, i32, P(i32)]),
        "hp_mbm_next": (i32, [v, P(i32), P(i32)]),
        "hp_mbm_destroy": (None, [v]),
        "hp_layernorm": (i32, [v, i64, i64, i64, v, v, v, i64, v]),
        "hp_embed": (i32, [v, i32, i32, i32, i32, v, v, i64, i64, i64, v, v]),
        "hp_attention_prefill": (i32, [v, i32, i32, i64, i32, v, v, v, i32, i32, v]),
        "hp_attention_decode_workspace_bytes": (C.c_size_t, [i32, i64, i32, i32]),
        "hp_attention_decode": (i32, [v, i32, i64, i32, i32, v, v, v, i32, i32, i32, v, C.c_size_t, v]),
        "hp_argmax": (i32, [v, i64, i32, i64, v, v]),
    })
    optional = {}
    for name, (res, args) in list(sig.items()) + list(optional.items()):
        if not hasattr(lib, name):
            if name in sig:
                raise ImportError(f"{LIB_PATH} does not export {name}")
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

EXPORTED = [
    "hp_last_error", "hp_abi_version", "hp_device_ok", "hp_packed_bytes", "hp_scale_count",
    "hp_quant_pack", "hp_quant_pack_stats", "hp_quant_unpack", "hp_dequant", "hp_indicator_stats",
    "hp_qlinear_workspace_bytes", "hp_qlinear", "hp_host_scaling_factor", "hp_host_g_of_x",
    "hp_host_indicator_csv", "hp_host_omega_from_stats", "hp_host_mc_output_variance", "hp_host_memcost", "hp_host_preset",
    "hp_host_make_schedule", "hp_host_simulate", "hp_host_plan_check", "hp_host_unit_order", "hp_host_latency_fit", "hp_host_latency_predict", "hp_set_sm_budget", "hp_set_pdl",
    "hp_nccl_unique_id", "hp_pipeline_create", "hp_pipeline_run", "hp_pipeline_stage_costs",
    "hp_pipeline_kernel_stats", "hp_pipeline_layer_costs", "hp_pipeline_info", "hp_pipeline_destroy",
    "hp_layernorm", "hp_embed", "hp_attention_prefill", "hp_attention_decode", "hp_attention_decode_workspace_bytes", "hp_argmax",
    "hp_pipeline_final_hidden", "hp_pipeline_load_stats", "hp_mbm_create", "hp_mbm_prefill_done",
    "hp_mbm_decode_done", "hp_mbm_next", "hp_mbm_destroy",
]


def check(status: int) -> None:
    if status == HP_OK:
        return
    msg = (lib.hp_last_error() or b"").decode(errors="replace")
    if status == HP_EINVAL:
        raise InvalidArgument(status, msg)
    if status == HP_EINFEASIBLE:
        raise Infeasible(status, msg)
    raise HPError(status, msg)


def device_ok() -> bool:
    return bool(lib.hp_device_ok())
