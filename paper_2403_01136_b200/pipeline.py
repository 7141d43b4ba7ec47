"""Python handle on the C++ pipeline executor (hp_pipeline_* in the C-ABI).

One process per GPU (torchrun); rank 0 creates one ncclUniqueId per
directed link and the caller broadcasts them (torch.distributed is only the
rendezvous — all activation traffic is NCCL P2P issued by the C++ runtime).
"""
from __future__ import annotations

import ctypes as C
import os
import json
from dataclasses import dataclass
from pathlib import Path

from . import capi
from .capi import check, lib

# The executor caps NCCL P2P channels at 2 per link (pipeline.cpp, only for
# world > 1 and only if the caller has not set NCCL_MAX_P2P_NCHANNELS). NCCL
# reads it at its first initialisation in the process, so a host that
# creates NCCL communicators before the Pipeline (torch.distributed with the
# nccl backend) sets it itself -- bench.py does; importing this module does
# not touch the environment.

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


class WeightSet:
    """Checkpoint sources for Pipeline(weights=...): per tensor a bf16 host
    buffer (anything exposing a data pointer: a pinned/pageable torch CPU
    tensor or a numpy array; kept alive here) or (path, byte offset) of a raw
    bf16 file. Missing entries are the seeded synthetic tensors."""

    def __init__(self, n_layers: int, bin_bytes: int = 0):
        self.n_layers = n_layers
        self.linear = [None] * (4 * n_layers)
        self.norm = [None] * (4 * n_layers)
        self.embed = self.pos = None
        self.final_norm = [None, None]
        self.bin_bytes = bin_bytes
        self._keep = []

    def _src(self, v):
        s = capi.hp_tensor_src()
        if v is None:
            return s
        if isinstance(v, tuple):  # (path, offset)
            path = str(v[0]).encode()
            self._keep.append(path)
            s.path, s.offset = path, int(v[1])
            return s
        self._keep.append(v)
        s.host = v.data_ptr() if hasattr(v, "data_ptr") else v.ctypes.data
        return s

    def c(self) -> capi.hp_weight_set:
        w = capi.hp_weight_set()
        w.n_layers = self.n_layers
        lin = (capi.hp_tensor_src * len(self.linear))(*[self._src(v) for v in self.linear])
        nrm = (capi.hp_tensor_src * len(self.norm))(*[self._src(v) for v in self.norm])
        self._keep += [lin, nrm]
        w.linear, w.norm = lin, nrm
        w.embed, w.pos = self._src(self.embed), self._src(self.pos)
        w.final_norm[0], w.final_norm[1] = self._src(self.final_norm[0]), self._src(self.final_norm[1])
        w.bin_bytes = self.bin_bytes
        return w


class Pipeline:
    def __init__(self, plan_json: str, model_json: str, rank: int = 0, world: int = 1,
                 ids: bytes | None = None, scheme: int = capi.HP_SYMMETRIC,
                 use_graphs: bool = True, instrument: bool = False, sm_budget: int = 0,
                 seed: int = 2403, weight_std: float = 0.02, timeout_s: float | None = None,
                 weights: WeightSet | None = None):
        if timeout_s is None:  # watchdog: a round stuck this long raises instead of hanging
            timeout_s = float(os.environ.get("HP_PIPELINE_TIMEOUT_S", "0"))
        opt = capi.hp_pipeline_options(scheme, int(use_graphs), int(instrument), sm_budget,
                                       seed, weight_std, timeout_s)
        h = C.c_void_p()
        idbuf = C.create_string_buffer(ids, len(ids)) if ids else None
        wc = weights.c() if weights is not None else None
        check(lib.hp_pipeline_create(plan_json.encode(), model_json.encode(), rank, world,
                                     idbuf, C.byref(opt), C.byref(wc) if wc is not None else None,
                                     C.byref(h)))
        self._h = h
        self.rank, self.world = rank, world
        self.plan = json.loads(plan_json)

    def run(self, host_tokens: int | None = None, host_out: int | None = None) -> Timing:
        """One round; host_tokens (rank 0): pointer to [B x s] int32 prompt ids
        (None: the synthetic prompt); host_out (last rank): [B x n] int32."""
        t = (C.c_double * 4)()
        check(lib.hp_pipeline_run(self._h, host_tokens, host_out, t))
        return Timing(*t)

    def final_hidden(self, host_ptr: int) -> None:
        check(lib.hp_pipeline_final_hidden(self._h, host_ptr))

    def load_stats(self):
        out = (C.c_double * 4)()
        check(lib.hp_pipeline_load_stats(self._h, out))
        return {"seconds": out[0], "source_bytes": out[1], "resident_bytes": out[2],
                "bins": int(out[3])}

    def stage_cost(self):
        out = (C.c_double * 4)()
        check(lib.hp_pipeline_stage_costs(self._h, out))
        return list(out)

    def kernel_stats(self, kind: int):
        """kind 0 prefill linear (K4), 1 decode linear (K3), 2 prefill
        attention, 3 decode attention."""
        out = (C.c_double * 4)()
        check(lib.hp_pipeline_kernel_stats(self._h, kind, out))
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
