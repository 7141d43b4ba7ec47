"""Closed-loop check of a plan: predict one serving
round of `plan` from its latency model (the planner's input: latcost
features, latcost.cpp:60-67, summed per stage and fed to pipesim::simulate,
pipesim.cpp:200-248) and compare with the round the B200 executor actually
runs.

  python tools/plan_eval.py opt30b_b32_1gpu_b200lat [more plans]   # 1-stage plans, 1 GPU

Prints one JSON line per plan: predicted vs measured makespan and their
relative error, plus the measured per-unit stage costs.
"""
from __future__ import annotations

import ctypes as C
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
PLANS = ROOT / "tests" / "golden" / "plans"


def predict(plan: dict, lat: dict) -> dict:
    from paper_2403_01136_b200 import capi
    dev = plan["devices"][0]
    w = plan["workload"]
    B, s, n, eta, xi = w["global_bz"], w["s"], w["n"], plan["eta"], plan["xi"]
    costs = []
    for j, st in enumerate(plan["stages"]):
        pre = dec = 0.0
        for l in range(*st["layers"]):
            c = lat[st.get("device", dev)][str(plan["layer_bits"][l])]
            f = [1, eta, s, eta * s, eta * s * s]
            pre += max(0.0, sum(a * b for a, b in zip(c["prefill"], f)))
            ts = range(1, n)
            dec += statistics.mean(max(0.0, sum(a * b for a, b in zip(c["decode"], [1, xi, xi * (t + s), t + s])))
                                   for t in ts)
        costs += [pre, dec, 0.0, 0.0]
    S = len(plan["stages"])
    arr = (C.c_double * len(costs))(*costs)
    out = (C.c_double * 4)()
    busy = (C.c_double * S)()
    capi.check(capi.lib.hp_host_simulate(arr, S, B, eta, xi, n, out, busy, None, 0))
    return {"makespan_s": out[0], "stage_costs_s": [[costs[4 * j], costs[4 * j + 1]] for j in range(S)]}


def main():
    from paper_2403_01136_b200.pipeline import Pipeline, load_plan
    for name in sys.argv[1:]:
        plan_json, model_json = load_plan(name)
        plan = json.loads(plan_json)
        lat = json.loads((PLANS / f"{name}.latency.json").read_text())
        pred = predict(plan, lat)
        p = Pipeline(plan_json, model_json)
        for _ in range(2):
            p.run()
        ts = [p.run().makespan_s for _ in range(3)]
        meas = statistics.median(ts)
        cost = p.stage_cost()
        p.close()
        print(json.dumps({"plan": name, "layer_bits": plan["layer_bits"], "eta": plan["eta"],
                          "xi": plan["xi"], "predicted_makespan_s": pred["makespan_s"],
                          "measured_makespan_s": meas,
                          "rel_err": abs(pred["makespan_s"] - meas) / meas,
                          "predicted_stage_costs_s": pred["stage_costs_s"],
                          "measured_unit_costs_s": cost[:2],
                          "objective_total": plan["objective"]["total"]}), flush=True)


if __name__ == "__main__":
    main()
