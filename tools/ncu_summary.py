"""Summarise ncu output of `bench.py` into profiles/ (run here, no GPU).

  launches <launches.csv> <out.json> [plan]
      per-kernel-class device time / count / share of the timed round from
      `ncu --metrics gpu__time_duration.sum --clock-control none
       --profile-from-start off --csv --log-file launches.csv python bench.py ...`
      (bench.py brackets its timed rounds with cudaProfilerStart/Stop).
  traffic <rep.ncu-rep> <k3|k4> <plan> [--layer L] [--out profiles/ncu_traffic.json]
      DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of
      the first 4 matching qgemm launches of the timed round -- layer 0's
      qkv/out/fc1/fc2 of the first decode (k3) or prefill (k4) unit -- next
      to their algorithmic bytes (pipeline.cpp k3_bytes).
"""
import csv
import io
import json
import math
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PLANS = ROOT / "tests" / "golden" / "plans"
# (h1, h2) of the reference presets (config.cpp model table)
PRESET_H = {"opt-125m": (768, 3072), "opt-1.3b": (2048, 8192), "opt-13b": (5120, 20480),
            "opt-30b": (7168, 28672), "opt-66b": (9216, 36864), "bloom-176b": (14336, 57344)}


def kernel_class(name: str) -> str:
    if "qgemm_kernel<" in name:
        bn = int(name.split("qgemm_kernel<")[1].split(",")[2])
        return "K3 decode qgemm (BN<=64)" if bn <= 64 else "K4 prefill qgemm (BN>=128)"
    for key, cls in (("layernorm", "layernorm (glue)"), ("gather_rows", "gather_rows (glue)"),
                     ("attn_prefill", "attention prefill (glue)"), ("attn_decode", "attention decode (glue)"),
                     ("embed_kernel", "embedding (glue)"), ("argmax", "argmax (glue)"),
                     ("nccl", "NCCL"), ("quant_pack", "K1 quant_pack"), ("stats_kernel", "K2 stats")):
        if key in name.lower():
            return cls
    return "other: " + name.split("(")[0][:60]


def rows_of(text: str):
    lines = [l for l in text.splitlines() if l.startswith('"')]
    return list(csv.DictReader(io.StringIO("\n".join(lines))))


def round_counts(plan_name: str):
    """Launches per class in ONE full round of the plan on one stage (the
    executor's forward: per layer 2 LN + 4 qgemm + 1 attention; per unit an
    embedding on stage 0 and gather + final LN + LM-head qgemm + argmax on the
    last stage -- the LM head is a BN<=64 qgemm, counted with K3)."""
    plan = json.loads((PLANS / f"{plan_name}.json").read_text())
    B, n = plan["workload"]["global_bz"], plan["workload"]["n"]
    eta, xi = plan["eta"], plan["xi"]
    layers = len(plan["layer_bits"])
    pre_units = -(-B // eta)
    dec_units = -(-B // xi) * (n - 1)
    units = pre_units + dec_units
    return {"K4 prefill qgemm (BN>=128)": 4 * layers * pre_units,
            "K3 decode qgemm (BN<=64)": 4 * layers * dec_units + units,
            "layernorm prefill (glue)": 2 * layers * pre_units + pre_units,
            "layernorm decode (glue)": 2 * layers * dec_units + dec_units,
            "attention prefill (glue)": layers * pre_units,
            "attention decode (glue)": layers * dec_units,
            "embedding (glue)": units, "argmax (glue)": units,
            "gather_rows (glue)": units}


def launches(path: str, out: str, plan_name: str | None = None) -> None:
    rows = rows_of(Path(path).read_text())
    per = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        s = v * {"ns": 1e-9, "nsecond": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3,
                   "ms": 1e-3}.get(unit, 1e-9)
        c = kernel_class(r["Kernel Name"])
        if c.startswith("layernorm"):  # one CTA per row: decode grid = group size
            rows_ln = int(r["Grid Size"].strip("()").split(",")[0])
            c = "layernorm decode (glue)" if rows_ln <= 256 else "layernorm prefill (glue)"
        per[c][0] += 1
        per[c][1] += s
        total += s
    res = {"source": Path(path).name, "launches": sum(v[0] for v in per.values()),
           "device_time_s": total,
           "note": "ncu per-launch times are serialised and cold-cache: compare shares, not absolutes",
           "classes": {c: {"launches": n, "time_s": t, "share": t / total if total else None}
                       for c, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1])}}
    if plan_name:
        # the window may hold part of a round; each class repeats identical
        # shapes, so round time per class = full-round launches x window mean
        cnt = round_counts(plan_name)
        est = {c: cnt[c] * per[c][1] / per[c][0] for c in cnt if per[c][0]}
        tot = sum(est.values())
        pre = sum(v for c, v in est.items() if "prefill" in c or "gather" in c)
        res["round_extrapolation"] = {
            "plan": plan_name, "round_launches": cnt,
            "classes": {c: {"mean_launch_s": per[c][1] / per[c][0], "round_time_s": v,
                            "share": v / tot} for c, v in est.items()},
            "prefill_share": pre / tot, "decode_share": 1 - pre / tot}
    Path(out).write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res, indent=1))


def alg_bytes(plan_name: str, kind: str, layer: int = 0):
    plan = json.loads((PLANS / f"{plan_name}.json").read_text())
    model = json.loads((PLANS / f"{plan_name}.config.json").read_text())["model"]
    h1, h2 = (model["h1"], model["h2"]) if "h1" in model else PRESET_H[model["preset"]]
    bits = plan["layer_bits"][layer]
    scheme = 1
    if kind == "k3":
        m = min(plan["xi"], plan["workload"]["global_bz"])
    else:
        m = min(plan["eta"], plan["workload"]["global_bz"]) * plan["workload"]["s"]
    out = []
    for n, k in ((3 * h1, h1), (h1, h1), (h2, h1), (h1, h2)):
        w = n * k
        b = 2.0 * w if bits == 16 else math.ceil(w * bits / 8) + 4.0 * w / 128 * (2 if scheme == 0 else 1)
        out.append({"n": n, "k": k, "bits": bits, "m": m, "alg_bytes": b + 2.0 * m * (k + n),
                    "flops": 2.0 * m * n * k})
    return out


def traffic(rep: str, kind: str, plan_name: str, out: str, layer: int = 0) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = [r for r in rows_of(raw) if r.get("ID", "").isdigit()]
    ops = alg_bytes(plan_name, kind, layer)
    got = []
    for r, op in zip(rows[:4], ops):
        rd = float(r["dram__bytes_read.sum"].replace(",", ""))
        wr = float(r["dram__bytes_write.sum"].replace(",", ""))
        got.append({"kernel": r["Kernel Name"][:60], "grid": r["Grid Size"], **op,
                    "dram_read": rd, "dram_write": wr,
                    "duration_ns": float(r["gpu__time_duration.sum"].replace(",", ""))})
    # ncu raw page reports units in the second header row: normalise to bytes
    units = rows_of(raw)[0]
    scale_r = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units.get("dram__bytes_read.sum", "byte"), 1)
    scale_w = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units.get("dram__bytes_write.sum", "byte"), 1)
    tscale = {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(units.get("gpu__time_duration.sum", "nsecond"), 1)
    for g in got:
        g["dram_read"] *= scale_r
        g["dram_write"] *= scale_w
        g["duration_ns"] *= tscale
        g["traffic_over_alg"] = (g["dram_read"] + g["dram_write"]) / g["alg_bytes"]
    entry = {"source": f"profiles/{Path(rep).stem}.ncu-rep (ncu --set full, bench.py timed round, layer {layer})",
             "launches": len(got),
             "dram_bytes_per_launch": sum(g["dram_read"] + g["dram_write"] for g in got) / len(got),
             "alg_bytes_per_launch": sum(g["alg_bytes"] for g in got) / len(got),
             "per_launch": got}
    p = Path(out)
    doc = json.loads(p.read_text()) if p.exists() else {}
    doc.setdefault(plan_name, {})[kind] = entry
    p.write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(entry, indent=1))


if __name__ == "__main__":
    a = sys.argv[1:]
    if a[0] == "launches":
        launches(a[1], a[2], a[3] if len(a) > 3 else None)
    elif a[0] == "traffic":
        out = a[a.index("--out") + 1] if "--out" in a else str(ROOT / "profiles" / "ncu_traffic.json")
        layer = int(a[a.index("--layer") + 1]) if "--layer" in a else 0
        traffic(a[1], a[2], a[3], out, layer)
    else:
        sys.exit(__doc__)
