"""Python handle on the C++ pipeline executor (hp_pipeline_* in the C-ABI).

One process per GPU (torchrun); rank 0 creates one ncclUniqueId per
directed link and the caller broadcasts them (torch.distributed is only the
rendezvous — all activation traffic is NCCL P2P issued by the C++ runtime).
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass
from pathlib import Path

from . import capi
from .capi import check, lib

# NCCL caches its parameters when it first initialises in the process: set
# the executor's P2P channel cap (pipeline.cpp build()) before anything --
# e.g. torch.distributed with the nccl backend -- creates a communicator.
os.environ.setdefault("NCCL_MAX_P2P_NCHANNELS", "2")

ROOT = Path(__file__).resolve().parents[1]
PLANS = ROOT / "tests" / "golden" / "plans"


def load_plan(name: str) -> tuple[str, str]:
    """(plan JSON text, model JSON text) of a committed plan fixture."""
    plan = (PLANS / f"{name}.json").read_text()
    cfg = json.loads((PLANS / f"{name}.config.json").read_text())
    return plan, json.dumps(cfg["model"])


def nccl_ids(world: int) -> bytes:
    buf = C.create_string_buffer(128 * world)
    for l in range(world):
        check(lib.hp_nccl_unique_id(C.byref(buf, 128 * l)))
    return buf.raw


@dataclass
class Timing:
    makespan_s: float
    prefill_s: float
    decode_s: float
    io_s: float


class Pipeline:
    def __init__(self, plan_json: str, model_json: str, rank: int = 0, world: int = 1,
                 ids: bytes | None = None, scheme: int = capi.HP_SYMMETRIC,
                 use_graphs: bool = True, instrument: bool = False, sm_budget: int = 0,
                 seed: int = 2403, weight_std: float = 0.02, timeout_s: float = 0.0,
                 decode_fused: bool = False):
        opt = capi.hp_pipeline_options(scheme, int(use_graphs), int(instrument), sm_budget,
                                       seed, weight_std, timeout_s, int(decode_fused))
        h = C.c_void_p()
        idbuf = C.create_string_buffer(ids, len(ids)) if ids else None
        check(lib.hp_pipeline_create(plan_json.encode(), model_json.encode(), rank, world,
                                     idbuf, C.byref(opt), C.byref(h)))
        self._h = h
        self.rank, self.world = rank, world
        self.plan = json.loads(plan_json)

    def run(self, host_in: int | None = None, host_out: int | None = None) -> Timing:
        t = (C.c_double * 4)()
        check(lib.hp_pipeline_run(self._h, host_in, host_out, t))
        return Timing(*t)

    def stage_cost(self):
        out = (C.c_double * 4)()
        check(lib.hp_pipeline_stage_costs(self._h, out))
        return list(out)

    def kernel_stats(self, phase: int):
        out = (C.c_double * 4)()
        check(lib.hp_pipeline_kernel_stats(self._h, phase, out))
        return {"launches": int(out[0]), "seconds": out[1], "bytes": out[2], "flops": out[3]}

    def layer_costs(self, phase: int) -> list[float]:
        n = C.c_int64()
        out = (C.c_double * 256)()
        check(lib.hp_pipeline_layer_costs(self._h, phase, out, 256, C.byref(n)))
        return list(out[:n.value])

    def info(self):
        out = (C.c_int64 * 4)()
        check(lib.hp_pipeline_info(self._h, out))
        return {"weight_bytes": out[0], "launches_per_round": out[1], "units": out[2],
                "layers": out[3]}

    def close(self):
        if self._h:
            lib.hp_pipeline_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
