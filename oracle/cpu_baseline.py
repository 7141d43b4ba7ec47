"""ORACLE / BASELINE INFRASTRUCTURE ONLY: the CPU arm of bench.py.

bench.py's `cpu_baseline` leg and its `--impl reference` arm call this
module; it imports NOTHING from the product package (paper_2403_01136_b200),
so the reference arm loads only oracle/*.so: libhp_oracle.so (the C
restatements) and, when present, oracle/_ref/libhetplan_ref.so (the
reference's own compiled code).

What is timed, on the host cores (SURVEY §8d "CPU baseline"):
  (ii) the layer forward of the adaptive-bitwidth linear path,
       y = x . (zero + (code - off) * step)^T (indicator.cpp:53) per op,
       blocked fp32 accumulate with OpenMP on all cores
       (hp_cpu_baseline.c). The reference has no layer forward,
       so this restatement is its CPU path ("port");
   - `sample_round`: a bounded, MEASURED sample of the bench workload -- one
     layer per distinct bit width of the plan, its 4 ops at m = xi (one
     decode group-token) and at a 128-token prefill chunk -- extrapolated to
     the plan's round (B*s prefill + B*(n-1) decode tokens over L layers);
   - `opt125m_full_round`: the whole BASELINE configs[0] round (OPT-125M,
     mixed 4/8 plan, B=8, s=512, n=100) run end to end, no extrapolation;
  (i)  the reference's own `quantize()` (indicator.cpp:19-56, oracle/_ref),
       single thread, per 128-group over sampled OPT-13B fc1 rows;
  (iii) the reference's `build_indicator_table` (indicator.cpp:113-127)
       on the plan's 40-layer stats.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import time
from pathlib import Path

import numpy as np

from . import port, ref, ref_available

PLANS = Path(__file__).resolve().parents[1] / "tests" / "golden" / "plans"
PRESETS = {"opt-13b": (40, 5120, 20480), "opt-30b": (48, 7168, 28672),
           "opt-66b": (64, 9216, 36864), "bloom-176b": (70, 14336, 57344)}


def load_plan(name: str) -> tuple[dict, dict]:
    plan = json.loads((PLANS / f"{name}.json").read_text())
    model = json.loads((PLANS / f"{name}.config.json").read_text())["model"]
    return plan, model


def dims(model: dict) -> tuple[int, int, int]:
    if "preset" in model:
        return PRESETS[model["preset"]]
    return model["num_layers"], model["h1"], model["h2"]


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class _Layer:
    """Packed-as-codes synthetic layer (values do not change the timing)."""

    def __init__(self, bits: int, h1: int, h2: int, rng):
        self.bits = bits
        self.ops = []
        for n, k in ((3 * h1, h1), (h1, h1), (h2, h1), (h1, h2)):
            G = -(-k // 128)
            # a random block tiled over the matrix: values do not change the timing
            if bits == 16:
                blk = (rng.standard_normal(1 << 16, dtype=np.float32) * 0.02).view(np.uint32)
                codes = np.resize((blk >> 16).astype(np.uint16), (n, k))
                st = None
            else:
                codes = np.resize(rng.integers(0, 1 << bits, 1 << 16, dtype=np.uint8), (n, k))
                st = np.full((n, G), 0.02 / (1 << (bits - 1)), dtype=np.float32)
            self.ops.append((codes, st, n, k))

    _x: dict = {}

    @classmethod
    def _input(cls, m: int, k: int, rng) -> np.ndarray:
        if (m, k) not in cls._x:
            blk = (rng.standard_normal(1 << 16, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)
            cls._x[(m, k)] = np.resize(blk, (m, k))
        return cls._x[(m, k)]

    def forward(self, m: int, nthreads: int, rng) -> float:
        """Wall time of the 4 ops on m tokens."""
        lib = port().lib
        dt = 0.0
        for codes, st, n, k in self.ops:
            x = self._input(m, k, rng)
            y = np.empty((m, n), dtype=np.float32)
            t0 = time.perf_counter()
            rc = lib.hpo_cpu_qlinear_f32(x.ctypes.data, m, k, codes.ctypes.data,
                                         st.ctypes.data if st is not None else None, None, n,
                                         self.bits, 1, y.ctypes.data, nthreads)
            dt += time.perf_counter() - t0
            assert rc == 0
        return dt


def _bind():
    lib = port().lib
    if not getattr(lib, "_hp_cpu_bound", False):
        lib.hpo_cpu_qlinear_f32.restype = C.c_int
        lib.hpo_cpu_qlinear_f32.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                            C.c_void_p, C.c_int]
        lib._hp_cpu_bound = True


class SampleRound:
    """One bounded measured sample per call (a bench "step" of the CPU arm)."""

    PREFILL_CHUNK = 128

    def __init__(self, plan: dict, model: dict, nthreads: int | None = None, seed: int = 0):
        _bind()
        self.plan, self.model = plan, model
        self.L, self.h1, self.h2 = dims(model)
        self.nthreads = nthreads or threads()
        self.rng = np.random.default_rng(seed)
        self.layers = {b: _Layer(b, self.h1, self.h2, self.rng) for b in sorted(set(plan["layer_bits"]))}

    def step(self) -> dict:
        t0 = time.perf_counter()
        xi = self.plan["xi"]
        t_dec = {b: L.forward(xi, self.nthreads, self.rng) for b, L in self.layers.items()}
        t_pre = {b: L.forward(self.PREFILL_CHUNK, self.nthreads, self.rng) for b, L in self.layers.items()}
        wall = time.perf_counter() - t0
        w = self.plan["workload"]
        B, s, n = w["global_bz"], w["s"], w["n"]
        groups = -(-B // xi)
        bits = self.plan["layer_bits"]
        dec_round = groups * (n - 1) * sum(t_dec[b] for b in bits)
        pre_round = (B * s / self.PREFILL_CHUNK) * sum(t_pre[b] for b in bits)
        tokens = B * s + B * (n - 1)
        sampled_flops = sum(2.0 * m * sum(nn * kk for _, _, nn, kk in L.ops)
                            for L in self.layers.values() for m in (xi, self.PREFILL_CHUNK))
        return {"value": tokens / (dec_round + pre_round), "unit": "tok/s",
                "sample_s": wall, "decode_tok_s": B * (n - 1) / dec_round,
                "prefill_tok_s": B * s / pre_round,
                "generated_tok_s": B * n / (dec_round + pre_round),
                "sample_gflop_s": sampled_flops / wall / 1e9,
                "sample": (f"measured: one layer per distinct bit width {sorted(self.layers)} of the "
                           f"plan [h1={self.h1}, h2={self.h2}], its 4 ops at m={xi} (decode "
                           f"group-token) and m={self.PREFILL_CHUNK} (prefill chunk), "
                           f"{wall:.2f} s; extrapolated to {self.L} layers x B={B}, s={s}, n={n} "
                           "(blocked fp32-accumulate OpenMP restatement of the dequant-GEMM, "
                           "oracle/hp_cpu_baseline.c)")}


def opt125m_full_round(nthreads: int | None = None) -> dict:
    """BASELINE configs[0] measured end to end on the CPU: OPT-125M, the
    reference planner's mixed 4/8 plan (opt125m_b8_1gpu), B=8, s=512, n=100,
    eta=1, xi=8: 8 prefill micro-batches of 512 tokens and 99 decode
    group-tokens of 8 through all 12 layers' 4 linear ops."""
    _bind()
    nthreads = nthreads or threads()
    plan, model = load_plan("opt125m_b8_1gpu")
    L, h1, h2 = dims(model)
    rng = np.random.default_rng(1)
    layers = [_Layer(b, h1, h2, rng) for b in plan["layer_bits"]]
    w = plan["workload"]
    B, s, n, eta, xi = w["global_bz"], w["s"], w["n"], plan["eta"], plan["xi"]
    t0 = time.perf_counter()
    pre = sum(Ly.forward(min(eta, B - k) * s, nthreads, rng) for k in range(0, B, eta) for Ly in layers)
    dec = sum(Ly.forward(min(xi, B - g), nthreads, rng)
              for g in range(0, B, xi) for _ in range(n - 1) for Ly in layers)
    wall = time.perf_counter() - t0
    tokens = B * s + B * (n - 1)
    return {"tok_s": tokens / (pre + dec), "round_s": pre + dec, "wall_s": wall,
            "prefill_tok_s": B * s / pre, "decode_tok_s": B * (n - 1) / dec,
            "generated_tok_s": B * n / (pre + dec), "cores": nthreads,
            "what": "OPT-125M opt125m_b8_1gpu round (BASELINE configs[0]), all 12 layers x 4 "
                    "linear ops, measured (no extrapolation)"}


def ref_quantize_rate(rows: int = 1024, k: int = 5120, bits: int = 4) -> dict | None:
    """(i) the reference's own quantize() (oracle/_ref, indicator.cpp:19-56),
    single thread, one call per 128-k group, over `rows` rows of an OPT-13B
    fc1-shaped bf16 weight."""
    if not ref_available():
        return None
    rng = np.random.default_rng(5)
    w = (rng.standard_normal((rows, k), dtype=np.float32) * 0.02).astype(np.float64)
    r = ref()
    t0 = time.perf_counter()
    for i in range(rows):
        for g in range(0, k, 128):
            r.quantize(w[i, g:g + 128], bits, 1)
    dt = time.perf_counter() - t0
    return {"mweights_per_s": rows * k / dt / 1e6, "weights": rows * k, "seconds": dt,
            "threads": 1, "what": f"reference quantize() per 128-group, {bits}-bit symmetric, "
                                  f"{rows} rows x {k} (OPT-13B fc1 rows), incl. ctypes call overhead"}


def ref_indicator_time(plan: dict, model: dict) -> dict | None:
    """(iii) the reference's build_indicator_table on an L-layer stats CSV."""
    if not ref_available():
        return None
    L, h1, h2 = dims(model)
    rows = ["layer,operator,d_w,w_min,w_max,x_mean,x_var"]
    for i in range(L):
        for o, (n, k) in zip(("qkv", "out", "fc1", "fc2"),
                             ((3 * h1, h1), (h1, h1), (h2, h1), (h1, h2))):
            rows.append(f"{i},{o},{n * k},-0.1,0.1,0.05,1.25")
    csv = "\n".join(rows) + "\n"
    r = ref()
    t0 = time.perf_counter()
    reps = 20
    for _ in range(reps):
        r.indicator_csv(csv, [3, 4, 8, 16], 1, 0)
    return {"seconds": (time.perf_counter() - t0) / reps, "layers": L,
            "what": "reference build_indicator_table (+ CSV parse/serialize), bits {3,4,8,16}"}
