"""Decode-step micro-benchmark: one decode step (xi tokens) through a stack of
OPT-shaped layers as the pipeline runs it (LN1, qkv, out+res, LN2,
fc1+relu, fc2+res per layer; per-op launches with PDL), captured in a CUDA
graph and CUDA-event timed; the stack's packed weights are >> L2.

  python tools/decode_step.py [--bits 16,16,8,4,...|3] [--h1 5120 --h2 20480] [--m 32]

Prints one JSON line: step time, algorithmic bytes (SURVEY §8d K3 bytes),
GB/s and the fraction of MEASURED_PEAKS hbm_gbs; --per-op also times every
op of one layer per distinct bit width in isolation (graph of 20 launches of
that op over 20 weight copies, > L2).
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

OPT13B_PLAN = [16, 16, 8, 4, 4, 4] + [3] * 27 + [4] * 7


def k3_bytes(n, k, bits, m, scheme=1):
    w = n * k
    b = 2 * w if bits == 16 else -(-w * bits // 8) + 4 * w // 128 * (2 if scheme == 0 else 1)
    return b + 2 * m * (n + k)


def main():
    import torch
    from paper_2403_01136_b200 import qweight
    from paper_2403_01136_b200.capi import check, lib
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", default=",".join(map(str, OPT13B_PLAN)))
    ap.add_argument("--layers", type=int, default=40)
    ap.add_argument("--h1", type=int, default=5120)
    ap.add_argument("--h2", type=int, default=20480)
    ap.add_argument("--m", type=int, default=32)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--per-op", action="store_true")
    ap.add_argument("--no-ln", action="store_true", help="timing experiment: skip the two LayerNorms")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    h1, h2, m = args.h1, args.h2, args.m
    bits = [int(b) for b in args.bits.split(",")]
    if len(bits) == 1:
        bits = bits * args.layers
    shapes = [(3 * h1, h1), (h1, h1), (h2, h1), (h1, h2)]
    layers, alg = [], 0
    for b in bits:
        ops = []
        for n, k in shapes:
            w = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
            ops.append(qweight.quantize(w, b))
            alg += k3_bytes(n, k, b, m)
            del w
        lns = [(torch.ones(h1, device=dev) if j % 2 == 0 else torch.zeros(h1, device=dev)).to(torch.bfloat16)
               for j in range(4)]
        layers.append((ops, lns))
    x0 = torch.randn(m, h1, device=dev).to(torch.bfloat16)
    a = torch.empty(m, h1, dtype=torch.bfloat16, device=dev)
    qkv = torch.empty(m, 3 * h1, dtype=torch.bfloat16, device=dev)
    f = torch.empty(m, h2, dtype=torch.bfloat16, device=dev)
    xp = x0.clone()

    def step():
        for ops, ln in layers:
            if not args.no_ln:
                check(lib.hp_layernorm(xp.data_ptr(), h1, m, h1, ln[0].data_ptr(), ln[1].data_ptr(),
                                       a.data_ptr(), h1, torch.cuda.current_stream().cuda_stream))
            qweight.qlinear(ops[0], a, out=qkv)
            qweight.qlinear(ops[1], qkv[:, 2 * h1:], out=xp, residual=xp)
            if not args.no_ln:
                check(lib.hp_layernorm(xp.data_ptr(), h1, m, h1, ln[2].data_ptr(), ln[3].data_ptr(),
                                       a.data_ptr(), h1, torch.cuda.current_stream().cuda_stream))
            qweight.qlinear(ops[2], a, out=f, relu=True)
            qweight.qlinear(ops[3], f, out=xp, residual=xp)

    def graph_time(fn):
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            fn()
            st.synchronize()
            with torch.cuda.graph(g, stream=st):
                fn()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        return sorted(ts)[len(ts) // 2]

    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {"hbm_gbs": 6528.7}
    t = graph_time(step)
    res = {"layers": len(bits), "h1": h1, "h2": h2, "m": m, "bits": args.bits,
           "step_us": t * 1e6, "us_per_layer": t * 1e6 / len(bits), "alg_MB": alg / 1e6,
           "GBs": alg / t / 1e9, "frac_hbm": alg / t / 1e9 / peaks["hbm_gbs"]}
    if args.per_op:
        ops_t = {}
        for b in sorted(set(bits)):
            for oi, (n, k) in enumerate(shapes):
                copies = [qweight.quantize((torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16), b)
                          for _ in range(max(2, min(20, (400 << 20) // max(1, k3_bytes(n, k, b, 0)))))]
                x = torch.randn(m, k, device=dev).to(torch.bfloat16)
                y = torch.empty(m, n, dtype=torch.bfloat16, device=dev)
                tt = graph_time(lambda: [qweight.qlinear(c, x, out=y) for c in copies]) / len(copies)
                ops_t[f"b{b}_{['qkv', 'out', 'fc1', 'fc2'][oi]}"] = {
                    "us": tt * 1e6, "GBs": k3_bytes(n, k, b, m) / tt / 1e9,
                    "ideal_us": k3_bytes(n, k, b, m) / peaks["hbm_gbs"] / 1e3}
                del copies
        res["per_op"] = ops_t
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
