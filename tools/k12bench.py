"""K1 (quantize + pack) and K2 (indicator statistics) micro-benchmark:
CUDA-event timed on the launching stream, L2 flushed (256 MB read) between
launches, achieved GB/s of ALGORITHMIC bytes against
MEASURED_PEAKS.json hbm_gbs.

  K1 bytes/op = K·N·2 (bf16 read) + ceil(K·N·b/8) (codes) + (K·N/128)·4 (scale)
                [+ (K·N/128)·4 zero, asymmetric]
  K2 bytes/op = K·N·2 (weights) + T·K·2 (calibration activations)

  python tools/k12bench.py [--shapes 20480x5120,...] [--bits 3,4,8] [--tokens 2048]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2403_01136_b200 import capi, qweight
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="15360x5120,5120x5120,20480x5120,5120x20480,57344x14336")
    ap.add_argument("--bits", default="3,4,8")
    ap.add_argument("--tokens", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()) \
        if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else {"hbm_gbs": 6650.0}
    hbm = peaks["hbm_gbs"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()

    def timed(fn):
        ts = []
        for i in range(args.reps + 2):
            flush.sum()  # read-only flush: no dirty lines leak into the timed launch
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(a.elapsed_time(b) * 1e-3)
        ts.sort()
        return ts[len(ts) // 2]

    rows = []
    for shp in args.shapes.split(","):
        n, k = map(int, shp.split("x"))
        w = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
        for b in map(int, args.bits.split(",")):
            for scheme in (capi.HP_SYMMETRIC, capi.HP_ASYMMETRIC):
                qw = qweight.quantize(w, b, scheme)
                nsc = int(capi.lib.hp_scale_count(n, k))

                def k1():
                    capi.check(capi.lib.hp_quant_pack(
                        w.data_ptr(), n, k, k, b, scheme, capi.HP_NEAREST, qw.packed.data_ptr(),
                        qw.scale.data_ptr(), qw.zero.data_ptr() if qw.zero is not None else None,
                        None, None, st.cuda_stream))
                t = timed(k1)
                by = n * k * 2 + qweight.packed_bytes(n, k, b) + nsc * 4 * (1 if scheme == capi.HP_SYMMETRIC else 2)
                rows.append({"kernel": "K1", "shape": [n, k], "bits": b,
                             "scheme": "sym" if scheme == capi.HP_SYMMETRIC else "asym",
                             "us": t * 1e6, "alg_bytes": by, "GBs": by / t / 1e9, "frac": by / t / 1e9 / hbm})
                print(json.dumps(rows[-1]), flush=True)
                if b == 4 and scheme == capi.HP_ASYMMETRIC:
                    # K1 with K2's weight min/max fused (hp_quant_pack_stats)
                    stt = torch.empty(5, dtype=torch.float64, device=dev)

                    def k1s():
                        capi.check(capi.lib.hp_quant_pack_stats(
                            w.data_ptr(), n, k, k, b, scheme, capi.HP_NEAREST, qw.packed.data_ptr(),
                            qw.scale.data_ptr(), qw.zero.data_ptr(), None, None, stt.data_ptr(),
                            st.cuda_stream))
                    t = timed(k1s)
                    rows.append({"kernel": "K1+stats", "shape": [n, k], "bits": b, "scheme": "asym",
                                 "us": t * 1e6, "alg_bytes": by, "GBs": by / t / 1e9,
                                 "frac": by / t / 1e9 / hbm})
                    print(json.dumps(rows[-1]), flush=True)
                del qw
        x = (torch.randn(args.tokens, k, device=dev) + 0.05).to(torch.bfloat16)
        out = torch.empty(5, dtype=torch.float64, device=dev)

        def k2():
            capi.check(capi.lib.hp_indicator_stats(w.data_ptr(), n, k, k, x.data_ptr(), args.tokens, k,
                                                   out.data_ptr(), st.cuda_stream))
        t = timed(k2)
        by = n * k * 2 + args.tokens * k * 2
        rows.append({"kernel": "K2", "shape": [n, k], "tokens": args.tokens, "us": t * 1e6,
                     "alg_bytes": by, "GBs": by / t / 1e9, "frac": by / t / 1e9 / hbm})
        print(json.dumps(rows[-1]), flush=True)

        def k2x():  # calibration part only: the weight part came from K1's fused pass
            capi.check(capi.lib.hp_indicator_stats(None, 0, k, 0, x.data_ptr(), args.tokens, k,
                                                   out.data_ptr(), st.cuda_stream))
        t = timed(k2x)
        by = args.tokens * k * 2
        rows.append({"kernel": "K2 (x only)", "shape": [n, k], "tokens": args.tokens, "us": t * 1e6,
                     "alg_bytes": by, "GBs": by / t / 1e9, "frac": by / t / 1e9 / hbm})
        print(json.dumps(rows[-1]), flush=True)
    print(json.dumps({"summary": True, "hbm_gbs": hbm,
                      "k1_best_frac": max(r["frac"] for r in rows if r["kernel"] == "K1"),
                      "k2_best_frac": max(r["frac"] for r in rows if r["kernel"] == "K2")}))  # noqa: E501


if __name__ == "__main__":
    main()
