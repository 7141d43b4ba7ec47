"""Profile per-layer costs of a 1-GPU plan on the B200.

    python tools/layer_costs.py [plan] [--out tests/golden/plans/b200_layer_costs.json]

Runs the plan through the pipeline executor with instrument=True and records,
for every layer, the device time (CUDA events, LN + 4 quantized linear ops)
of one prefill micro-batch (eta*s rows) and of one decode group-token (xi
rows) -- medians over rounds. tests/golden/make_plans.py partitions the
weak-scaled bench plans on these measured costs (LLM-PQ's profiled latency
model, paper §5)."""
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    args = sys.argv[1:]
    out = Path(args[args.index("--out") + 1]) if "--out" in args else \
        ROOT / "tests" / "golden" / "plans" / "b200_layer_costs.json"
    name = next((a for a in args if not a.startswith("--") and not a.endswith(".json")),
                "opt13b_b32_1gpu")
    from paper_2403_01136_b200.pipeline import Pipeline, load_plan
    plan_json, model_json = load_plan(name)
    plan = json.loads(plan_json)
    p = Pipeline(plan_json, model_json, instrument=True)
    for _ in range(3):
        p.run()
    pre, dec = [], []
    for _ in range(5):
        p.run()
        pre.append(p.layer_costs(0))
        dec.append(p.layer_costs(1))
    p.close()
    L = len(plan["layer_bits"])
    res = {"plan": name, "device": "b200", "eta": plan["eta"], "xi": plan["xi"],
           "s": plan["workload"]["s"], "layer_bits": plan["layer_bits"],
           "prefill_s": [statistics.median(r[i] for r in pre) for i in range(L)],
           "decode_s": [statistics.median(r[i] for r in dec) for i in range(L)],
           "method": "CUDA events around each layer (LN + qkv/out/fc1/fc2) of one instrumented "
                     "prefill micro-batch and one decode group-token, graph-captured round, "
                     "median of 5 rounds (tools/layer_costs.py)"}
    out.write_text(json.dumps(res, indent=1) + "\n")
    by_bits = {}
    for b, ps, ds in zip(res["layer_bits"], res["prefill_s"], res["decode_s"]):
        by_bits.setdefault(b, []).append((ps, ds))
    for b, v in sorted(by_bits.items()):
        print(f"bits {b:2d}: {len(v):2d} layers, prefill {1e3 * statistics.mean(x[0] for x in v):.3f} ms,"
              f" decode {1e6 * statistics.mean(x[1] for x in v):.1f} us")


if __name__ == "__main__":
    main()
