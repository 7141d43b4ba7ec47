"""Plan fixtures from the REFERENCE planner (oracle/_ref; optimizer_planner.cpp
:79-170), one per BASELINE.json config. Run here (needs /root/reference):

    python tests/golden/make_plans.py [name ...]

Inputs: a roofline-derived synthetic B200 latency model
(latcost coefficient vectors, latcost.hpp:6-7), link 9e11 B/s, theta 0.001,
5 s per exact solve; omega for OPT-125M from the synthetic weights the B200
runtime generates (oracle/synth.py, stats through the oracle port), and the
SURVEY's synthetic omega_{i,b} = (8, 1.5, 0.005, 0)(1 + 0.01 i) for the large
shapes. Memory budgets are planning knobs that make the plans mixed-bit
(at 180 GB memory never binds). Writes tests/golden/plans/<name>.json plus
the omega CSV used.
"""
from __future__ import annotations

import json
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
OUT = Path(__file__).resolve().parent / "plans"
GiB = 1 << 30
FL, BW = 1.3486e15, 6.5456e12

MODELS = {
    "opt-125m": dict(name="opt-125m", num_layers=12, h1=768, h2=3072, num_heads=12,
                     vocab_s=50272, pos_s=2050),
    "opt-13b": {"preset": "opt-13b"}, "opt-30b": {"preset": "opt-30b"},
    "opt-66b": {"preset": "opt-66b"}, "bloom-176b": {"preset": "bloom-176b"},
}
SHAPES = {"opt-125m": (12, 768, 3072), "opt-13b": (40, 5120, 20480),
          "opt-30b": (48, 7168, 28672), "opt-66b": (64, 9216, 36864),
          "bloom-176b": (70, 14336, 57344)}

CONFIGS = {
    "opt125m_b8_1gpu": dict(model="opt-125m", devices=1, mem=400 * (1 << 20), B=8,
                            supported=[4, 8], group=1, omega="synthetic-weights"),
    "opt13b_b32_1gpu": dict(model="opt-13b", devices=1, mem=22 * GiB, B=32, supported=None,
                            group=1, omega="survey"),
    # north_star target: OPT-30B-shaped mixed 3/4/8/16 plan on ONE B200; the
    # 44 GiB budget (KV alone is 26.9 GB at B = 32) makes the plan mixed
    "opt30b_b32_1gpu": dict(model="opt-30b", devices=1, mem=44 * GiB, B=32, supported=None,
                            group=1, omega="survey"),
    # SURVEY §8f rank 1, the LLM-PQ loop closed on B200: the same configs
    # planned with the latency model FITTED on this build's kernels
    # (tools/latency_profile.py -> b200_<model>.latency_model.json)
    "opt13b_b32_1gpu_b200lat": dict(model="opt-13b", devices=1, mem=22 * GiB, B=32, supported=None,
                                    group=1, omega="survey", latency="b200_opt13b"),
    "opt30b_b32_1gpu_b200lat": dict(model="opt-30b", devices=1, mem=44 * GiB, B=32, supported=None,
                                    group=1, omega="survey", latency="b200_opt30b"),
    "opt66b_b32_8gpu_b200lat": dict(model="opt-66b", devices=8, mem=12 * GiB, B=32, supported=[4, 8],
                                    group=2, omega="survey", latency="b200_opt66b"),
    "bloom176b_b32_8gpu_b200lat": dict(model="bloom-176b", devices=8, mem=24 * GiB, B=32,
                                       supported=[3, 4, 8], group=2, omega="survey",
                                       latency="b200_bloom176b"),
    "opt30b_b32_2gpu": dict(model="opt-30b", devices=2, mem=24 * GiB, B=32, supported=None,
                            group=2, omega="survey"),
    "opt30b_b32_4gpu": dict(model="opt-30b", devices=4, mem=12 * GiB, B=32, supported=None,
                            group=2, omega="survey"),
    "opt66b_b32_8gpu": dict(model="opt-66b", devices=8, mem=12 * GiB, B=32, supported=[4, 8],
                            group=2, omega="survey"),
    "bloom176b_b32_8gpu": dict(model="bloom-176b", devices=8, mem=24 * GiB, B=32,
                               supported=[3, 4, 8], group=2, omega="survey"),
}


def latency_json(model: str) -> str:
    L, h1, h2 = SHAPES[model]
    P = 4 * h1 * h1 + 2 * h1 * h2
    per_bit = {}
    for b in (3, 4, 8, 16):
        eff = 1.0 if b == 16 else 0.8
        per_bit[str(b)] = {"prefill": [5e-6, 0.0, 0.0, 2 * P / (FL * eff), 4 * h1 / FL],
                           "decode": [5e-6 + P * b / 8 / BW, 0.0, 4 * h1 / BW, 0.0]}
    return json.dumps({"b200": per_bit})


def measured_latency_json(stem: str) -> str:
    """The fitted B200 model (latcost serialize_model format, from
    tools/latency_profile.py) in the planner input schema
    {device: {bit: {"prefill": [5], "decode": [4]}}}."""
    m = json.loads((OUT / f"{stem}.latency_model.json").read_text())
    out: dict = {}
    for g in m["groups"]:
        out.setdefault(g["device"], {}).setdefault(str(g["bit"]), {})[g["phase"]] = g["coeffs"]
    return json.dumps(out)


def omega_survey(L: int) -> str:
    rows = ["layer,bit_3,bit_4,bit_8,bit_16"]
    for i in range(L):
        f = 1 + 0.01 * i
        rows.append(f"{i},{8 * f!r},{1.5 * f!r},{0.005 * f!r},0")
    return "\n".join(rows) + "\n"


def omega_from_synthetic(model: str) -> str:
    """Stats of the runtime's synthetic weights / calibration activations,
    reduced by the oracle, omega by the reference build."""
    import oracle
    from oracle import synth
    L, h1, h2 = SHAPES[model]
    shapes = [(3 * h1, h1), (h1, h1), (h2, h1), (h1, h2)]
    sig2 = [1.0, 1.25, 1.5, 1.75]
    names = ["qkv", "out", "fc1", "fc2"]
    T = 256
    rows = ["layer,operator,d_w,w_min,w_max,x_mean,x_var"]
    for i in range(L):
        for o, ((n, k), s2) in enumerate(zip(shapes, sig2)):
            wb = synth.synth_bits(n * k, synth.seed_for(1, i, o), 0.0, 0.02)
            wf = (wb.astype(np.uint32) << 16).view(np.float32)
            xb = synth.synth_bits(T * k, synth.seed_for(2, i, o), 0.05, float(np.sqrt(s2)))
            mean, var = oracle.port().x_stats(xb)
            rows.append(f"{i},{names[o]},{n * k},{float(wf.min())!r},{float(wf.max())!r},"
                        f"{mean!r},{var!r}")
    stats = "\n".join(rows) + "\n"
    (OUT / f"{model}_calibration_stats.csv").write_text(stats)
    return oracle.ref().indicator_csv(stats, [3, 4, 8, 16], 1, 0)


def run(name: str) -> str:
    import oracle
    c = CONFIGS[name]
    L = SHAPES[c["model"]][0]
    omega = omega_from_synthetic(c["model"]) if c["omega"] == "synthetic-weights" else omega_survey(L)
    lat = (measured_latency_json(c["latency"]) if c.get("latency") else latency_json(c["model"]))
    dev = {"name": "b200", "mem_bytes": c["mem"], "link_bw_bytes_per_s": 9e11}
    if c["supported"]:
        dev["supported_bits"] = c["supported"]
    cfg = {"format_version": 1, "model": MODELS[c["model"]],
           "cluster": {"devices": [dev] * c["devices"]},
           "workload": {"B": c["B"], "s": 512, "n": 100}, "bits": [3, 4, 8, 16]}
    t0 = time.time()
    plan = oracle.ref().best_plan(json.dumps(cfg), omega, lat, 0.001,
                                  group=c["group"], heuristic=False, time_limit_s=5.0)
    dt = time.time() - t0
    doc = json.loads(plan)
    doc["_fixture"] = {"generator": "tests/golden/make_plans.py", "config": c,
                       "omega_source": c["omega"], "planner_seconds": round(dt, 1)}
    (OUT / f"{name}.json").write_text(json.dumps(doc, indent=1))
    (OUT / f"{name}.omega.csv").write_text(omega)
    (OUT / f"{name}.config.json").write_text(json.dumps(cfg, indent=1))
    (OUT / f"{name}.latency.json").write_text(lat)
    return f"{name}: {dt:.0f}s bits={doc['layer_bits']} stages={[s['layers'] for s in doc['stages']]} eta={doc['eta']} xi={doc['xi']} optimal={doc['optimal']}"


def weak(n_dev: int, base: str = "opt13b_b32_1gpu") -> str:
    """Weak-scaled pipeline plan for bench.py --gpus N: the configs[1] plan's
    bit assignment (same 40 layers, same bits) with B = 32 N requests, eta 4,
    xi 32 -- N decode groups in flight, so every stage has one group to work
    on -- and layers split into N contiguous stages minimising the maximum
    per-stage work of one round, 8N prefill micro-batches + 99N decode
    group-tokens, on the per-layer costs MEASURED on a B200
    (b200_layer_costs.json, tools/layer_costs.py). NOT a reference-planner output: the planner
    prefers xi = B (one decode group), which leaves a
    pipeline nothing to overlap in decode. The objective parts follow the
    same latency model and recompose exactly (types.cpp:17-24, :118-122)."""
    src = json.loads((OUT / f"{base}.json").read_text())
    bits = src["layer_bits"]
    L, h1, h2 = SHAPES[src["model"]]
    P = 4 * h1 * h1 + 2 * h1 * h2
    s, eta, xi = src["workload"]["s"], src["eta"], 32
    B = 32 * n_dev
    meas = json.loads((OUT / "b200_layer_costs.json").read_text())
    assert meas["layer_bits"] == bits and meas["eta"] == eta, "layer costs of another plan"
    pre, dec = meas["prefill_s"], meas["decode_s"]
    n_pre = -(-B // eta) // n_dev              # per-device-share of micro-batches
    n_dec = (src["workload"]["n"] - 1)         # group-tokens per group
    work = [n_pre * p_ + n_dec * d_ for p_, d_ in zip(pre, dec)]
    # contiguous min-max partition (DP over split points)
    INF = float("inf")
    pref = [0.0]
    for w_ in work:
        pref.append(pref[-1] + w_)
    best = [[INF] * (L + 1) for _ in range(n_dev + 1)]
    cut = [[0] * (L + 1) for _ in range(n_dev + 1)]
    best[0][0] = 0.0
    for j in range(1, n_dev + 1):
        for e in range(j, L + 1):
            for b0 in range(j - 1, e):
                v = max(best[j - 1][b0], pref[e] - pref[b0])
                if v < best[j][e]:
                    best[j][e], cut[j][e] = v, b0
    bounds, e = [], L
    for j in range(n_dev, 0, -1):
        bounds.append((cut[j][e], e))
        e = cut[j][e]
    bounds.reverse()
    t_pre = [sum(pre[a:b]) for a, b in bounds]
    t_dec = [sum(dec[a:b]) for a, b in bounds]
    omega = {int(r.split(",")[0]): [float(x) for x in r.split(",")[1:]]
             for r in (OUT / f"{base}.omega.csv").read_text().splitlines()[1:] if r}
    col = {3: 0, 4: 1, 8: 2, 16: 3}
    omega_sum = sum(omega[i][col[b]] for i, b in enumerate(bits))
    theta, n = src["theta"], src["workload"]["n"]
    bc = lambda u: -(-(B - u) // u)
    obj = {"t_max_pre": max(t_pre), "t_max_dec": max(t_dec), "t_pre_total": sum(t_pre),
           "t_dec_total": sum(t_dec), "omega_sum": omega_sum, "theta": theta}
    obj["total"] = (bc(eta) * obj["t_max_pre"] + bc(xi) * (n - 1) * obj["t_max_dec"]
                    + obj["t_pre_total"] + obj["t_dec_total"] + theta * omega_sum)
    name = f"opt13b_b{B}_{n_dev}gpu_weak"
    doc = dict(src)
    doc.update({"workload": {"global_bz": B, "s": s, "n": n}, "eta": eta, "xi": xi,
                "device_order": list(range(n_dev)), "devices": ["b200"] * n_dev,
                "stages": [{"device_index": j, "device": "b200", "layers": [a, b]}
                           for j, (a, b) in enumerate(bounds)],
                "objective": obj, "optimal": False})
    doc["_fixture"] = {"generator": "tests/golden/make_plans.py weak", "derived_from": base,
                       "note": weak.__doc__.split("\n\n")[0]}
    cfg = json.loads((OUT / f"{base}.config.json").read_text())
    cfg["cluster"]["devices"] = [cfg["cluster"]["devices"][0]] * n_dev
    cfg["workload"]["B"] = B
    (OUT / f"{name}.json").write_text(json.dumps(doc, indent=1))
    (OUT / f"{name}.config.json").write_text(json.dumps(cfg, indent=1))
    (OUT / f"{name}.omega.csv").write_text((OUT / f"{base}.omega.csv").read_text())
    (OUT / f"{name}.latency.json").write_text((OUT / f"{base}.latency.json").read_text())
    return (f"{name}: stages={bounds} work/stage="
            f"{[round(n_dev * (pref[b] - pref[a]), 3) for a, b in bounds]} s")


if __name__ == "__main__":
    OUT.mkdir(exist_ok=True)
    if sys.argv[1:2] == ["weak"]:
        for nd in (2, 4, 8):
            print(weak(nd))
        sys.exit(0)
    names = sys.argv[1:] or list(CONFIGS)
    with ProcessPoolExecutor(max_workers=min(len(names), 6)) as ex:
        for line in ex.map(run, names):
            print(line, flush=True)
