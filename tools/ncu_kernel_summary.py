"""Compact per-launch summary of `ncu --set full` captures (run here, no GPU).

  python tools/ncu_kernel_summary.py OUT.json NAME=REP.ncu-rep[:ALG_BYTES] ...

For every launch in each report: duration, DRAM bytes read/written, DRAM
GB/s, SM throughput, IPC, issue-slot utilisation, occupancy and the top warp
stall reasons; with ALG_BYTES (the kernel's algorithmic bytes per launch,
SURVEY §8d / DESIGN.md §4) also achieved algorithmic GB/s, its fraction of
MEASURED_PEAKS.json hbm_gbs and traffic / algorithmic bytes.
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return [dict(zip(hdr, r)) for r in data], dict(zip(hdr, units))


def num(d, k, unit_scale=None):
    v = d.get(k, "")
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def scaled(d, units, k):
    """Value converted to base units (bytes, seconds) from ncu's display unit."""
    v = num(d, k)
    if v is None:
        return None
    u = units.get(k, "")
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
            "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
            "ms": 1e-3}.get(u, 1.0)
    return v * mult


def main():
    out = Path(sys.argv[1])
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = peaks.get("hbm_gbs", 6545.6)
    res = {"hbm_gbs_peak": hbm, "source": "ncu --set full --clock-control none (tools/gpu/*.sh)", "kernels": {}}
    for arg in sys.argv[2:]:
        name, spec = arg.split("=", 1)
        rep, _, alg = spec.partition(":")
        launches, units = raw(rep)
        items = []
        for d in launches:
            t = scaled(d, units, "gpu__time_duration.sum")
            rd = scaled(d, units, "dram__bytes_read.sum")
            wr = scaled(d, units, "dram__bytes_write.sum")
            stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""):
                      num(d, k) for k in d if k.startswith("smsp__average_warps_issue_stalled_")
                      and k.endswith("_per_issue_active.ratio")}
            top = sorted(((k, v) for k, v in stalls.items() if v), key=lambda kv: -kv[1])[:5]
            e = {"kernel": d.get("Kernel Name", "")[:120], "grid": d.get("launch__grid_size"),
                 "block": d.get("launch__block_size"), "registers": d.get("launch__registers_per_thread"),
                 "duration_us": t * 1e6 if t else None, "dram_read": rd, "dram_write": wr,
                 "dram_GBs": (rd + wr) / t / 1e9 if t and rd is not None and wr is not None else None,
                 "sm_throughput_pct": num(d, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                 "ipc_active": num(d, "sm__inst_executed.avg.per_cycle_active"),
                 "issue_slots_busy_pct": num(d, "sm__inst_issued.avg.pct_of_peak_sustained_active"),
                 "warps_active_pct": num(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
                 "top_stalls_per_issue": dict(top)}
            if alg and t:
                a = float(alg)
                e.update({"alg_bytes": a, "alg_GBs": a / t / 1e9, "frac_of_hbm_peak": a / t / 1e9 / hbm,
                          "traffic_over_alg": (rd + wr) / a if rd is not None and wr is not None else None})
            items.append(e)
        res["kernels"][name] = {"report": rep, "launches": items}
    out.write_text(json.dumps(res, indent=1))
    for n, k in res["kernels"].items():
        for e in k["launches"]:
            print(n, {kk: (round(v, 3) if isinstance(v, float) else v) for kk, v in e.items()
                      if kk in ("duration_us", "dram_GBs", "alg_GBs", "frac_of_hbm_peak", "ipc_active",
                                "issue_slots_busy_pct", "traffic_over_alg")})


if __name__ == "__main__":
    main()
