"""Generate the golden fixtures of the adaptive-bitwidth linear path from
the REFERENCE'S OWN CODE (oracle/_ref/libhetplan_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile). Run here, where
/root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

Outputs (committed, small): tests/golden/quant_golden.npz,
tests/golden/planning_golden.json. The GPU box never reads /root/reference;
the tests compare against these files and the oracle port.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent


def to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """float -> bf16 bit patterns, round-to-nearest-even (as torch does)."""
    f = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounding = ((f >> 16) & 1) + 0x7FFF
    return ((f + rounding) >> 16).astype(np.uint16)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def vectors(rng):
    """Named bf16-valued test vectors: SPEC / SURVEY App. C known answers,
    ties, ragged lengths, flat groups, outliers."""
    v = {
        "appc_row1": [-3, -2.5, -1.5, -0.5, 0.5, 1.5, 2.5, 3],
        "appc_row2": [-0.5, -0.25, 0, 0.125, 0.3125, 0.4375, 0.5, 1.0],
        "flat_pos": [0.25] * 4,
        "flat_zero": [0.0] * 16,
        "single": [0.75],
        "two": [-1.0, 1.0],
        "spec_asym_255": list(np.linspace(0, 2.55, 52)),
    }
    for n in (5, 127, 128):
        v[f"normal_{n}"] = list(rng.normal(0, 0.02, n))
    w = rng.normal(0, 0.02, 128)
    w[rng.integers(0, 128, 3)] *= 8.0  # outliers exercise the clamp/range
    v["outliers_128"] = list(w)
    # exact-tie heavy: small integers / 2
    v["ties_128"] = list(rng.integers(-40, 41, 128) / 8.0)
    out = {}
    for k, arr in v.items():
        out[k] = bf16_bits_to_f64(to_bf16_bits(np.array(arr, dtype=np.float64)))
    return out


def main():
    ref = oracle.ref()
    rng = np.random.default_rng(2403)
    arrays = {}
    # ---- per-vector quantize() golden (codes / step / zero) -----------------
    vecs = vectors(rng)
    for name, w in vecs.items():
        arrays[f"vec/{name}/w"] = w
        for bits in (3, 4, 8):
            for scheme in (0, 1):
                codes, step, zero = ref.quantize_codes(w, bits, scheme)
                arrays[f"vec/{name}/b{bits}s{scheme}/codes"] = codes
                arrays[f"vec/{name}/b{bits}s{scheme}/stepzero"] = np.array([step, zero])
                arrays[f"vec/{name}/b{bits}s{scheme}/out"] = ref.quantize(w, bits, scheme)
    # ---- matrix golden: group-wise over rows (aligned + ragged shapes) ------
    for (n, k, tag) in ((256, 384, "aligned"), (130, 200, "ragged")):
        wb = to_bf16_bits(rng.normal(0, 0.02, (n, k)))
        wb[3, 5] = to_bf16_bits(np.array([0.5]))[0]        # outlier
        wb[7, :] = to_bf16_bits(np.array([0.125]))[0]      # flat rows
        arrays[f"mat/{tag}/w_bits"] = wb
        wf = bf16_bits_to_f64(wb)
        G = -(-k // 128)
        for bits in (3, 4, 8):
            for scheme in (0, 1):
                off = (1 << (bits - 1)) - 1 if scheme == 1 else 0
                codes = np.zeros((n, k), dtype=np.uint8)
                step = np.zeros((n, G))
                zero = np.zeros((n, G))
                for r in range(n):
                    for g in range(G):
                        seg = wf[r, g * 128:(g + 1) * 128]
                        c, s, z = ref.quantize_codes(seg, bits, scheme)
                        codes[r, g * 128:g * 128 + len(seg)] = (c + off).astype(np.uint8)
                        step[r, g] = s
                        zero[r, g] = z
                arrays[f"mat/{tag}/b{bits}s{scheme}/codes"] = codes
                arrays[f"mat/{tag}/b{bits}s{scheme}/step"] = step
                arrays[f"mat/{tag}/b{bits}s{scheme}/zero"] = zero
    np.savez_compressed(OUT / "quant_golden.npz", **arrays)

    # ---- planning-side golden (indicator, memcost, schedule, simulate) ------
    g = {}
    calib = (Path("/root/reference/proj/data/sample_calibration.csv")).read_text()
    g["sample_calibration_csv"] = calib
    g["omega_sample_sym_nearest"] = ref.indicator_csv(calib, [3, 4, 8, 16], 1, 0)
    g["omega_sample_asym_stoch"] = ref.indicator_csv(calib, [2, 3, 4, 8, 16], 0, 1)
    # random stats table
    rows = ["layer,operator,d_w,w_min,w_max,x_mean,x_var"]
    for layer in range(6):
        for op, dw in (("qkv", 3 * 768 * 768), ("out", 768 * 768), ("fc1", 3072 * 768),
                       ("fc2", 768 * 3072)):
            lo = -abs(rng.normal(0.1, 0.03))
            hi = abs(rng.normal(0.1, 0.03))
            rows.append(f"{layer},{op},{dw},{lo!r},{hi!r},{rng.normal(0.05, 0.01)!r},"
                        f"{abs(rng.normal(1.2, 0.3))!r}")
    rand_csv = "\n".join(rows) + "\n"
    g["random_stats_csv"] = rand_csv
    g["omega_random_sym_nearest"] = ref.indicator_csv(rand_csv, [3, 4, 8, 16], 1, 0)
    g["scaling_factor"] = [[a, b, bit, s, ref.scaling_factor(a, b, bit, s)]
                           for a, b, bit, s in ((0.0, 2.55, 8, 0), (-7.0, 7.0, 4, 1),
                                                (-1.0, 1.0, 4, 1), (0.3, 0.3, 3, 0),
                                                (-0.05810546875, 0.07, 4, 0))]
    g["g_of_x"] = [[m, v, r, ref.g_of_x(m, v, r)] for m, v, r in
                   ((0.0, 1.0, 0), (0.0, 1.0, 1), (2.0, 1.0, 1), (0.05, 1.75, 0))]
    models = {name: ref.preset(name) for name in
              ("opt-13b", "opt-30b", "opt-66b", "bloom-176b", "tiny-test")}
    models["opt-125m"] = [12, 768, 3072, 12, 50272, 2050, 768, 768, 0]
    g["models"] = models
    g["memcost"] = {name: {str(bit): ref.memcost(f, bit, 32, 512, 100)
                           for bit in (2, 3, 4, 8, 16)} for name, f in models.items()}
    sched = []
    for B, eta, xi in ((8, 2, 4), (5, 2, 5), (8, 3, 6), (32, 2, 32), (32, 32, 32), (7, 1, 7),
                       (12, 5, 6), (1, 1, 1)):
        sched.append([B, eta, xi, *ref.make_schedule(B, eta, xi)])
    g["schedules"] = sched
    sims = []
    cases = [
        ([[1.5, 0.25, 0, 0]], 1, 1, 1, 11),
        ([[2, 0.1, 0, 0], [2, 0.1, 0, 0]], 4, 1, 4, 1),
        ([[2.0, 0.1, 0, 0], [2.0, 0.1, 0, 0]], 8, 2, 4, 11),
        ([[0.5, 0.01, 1e-3, 1e-4], [0.6, 0.012, 1e-3, 1e-4], [0.55, 0.011, 1e-3, 1e-4],
          [0.5, 0.01, 0, 0]], 32, 2, 32, 100),
        ([[0.3, 0.02, 0.05, 0.002], [0.2, 0.03, 0.0, 0.0]], 12, 5, 6, 7),
        ([[1e-3, 2e-4, 3e-4, 1e-5]] * 8, 32, 1, 32, 100),
    ]
    for costs, B, eta, xi, n in cases:
        r = ref.simulate(np.array(costs, dtype=np.float64), B, eta, xi, n, timeline=True)
        sims.append({"costs": costs, "B": B, "eta": eta, "xi": xi, "n": n,
                     "makespan": r["makespan"], "bubble": r["bubble"],
                     "analytic": r["analytic"], "busy": r["busy"],
                     "timeline_head": r["timeline"][:64].tolist(), "events": r["events"]})
    g["simulate"] = sims
    mc_w = [(i - 32) / 40 for i in range(64)]
    g["mc_output_variance"] = {
        "w": mc_w, "mean": 0.5, "var": 1.0, "bit": 4, "scheme": 1, "rounding": 1,
        "samples": 20000, "seed": 42,
        "result": ref.mc_output_variance(mc_w, 0.5, 1.0, 4, 1, 1, 20000, 42)}
    (OUT / "planning_golden.json").write_text(json.dumps(g, indent=1))
    print("wrote", OUT / "quant_golden.npz", OUT / "planning_golden.json")


if __name__ == "__main__":
    main()
