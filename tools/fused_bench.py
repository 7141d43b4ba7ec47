"""Decode-step micro-benchmark: one decode step (xi tokens) through a stack of
OPT-shaped layers, K3 fused (hp_decode_plan, one launch) vs the per-op
launches (hp_layernorm + hp_qlinear), CUDA-event timed, weights >> L2.

  python tools/fused_bench.py [--bits 16,16,8,4,...] [--h1 5120 --h2 20480] [--m 32]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

OPT13B_PLAN = [16, 16, 8, 4, 4, 4] + [3] * 27 + [4] * 7


def main():
    import torch
    from paper_2403_01136_b200 import qweight
    from paper_2403_01136_b200.capi import check, lib
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", default=",".join(map(str, OPT13B_PLAN)))
    ap.add_argument("--h1", type=int, default=5120)
    ap.add_argument("--h2", type=int, default=20480)
    ap.add_argument("--m", type=int, default=32)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--per-op", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    h1, h2, m = args.h1, args.h2, args.m
    bits = [int(b) for b in args.bits.split(",")]
    shapes = [(3 * h1, h1), (h1, h1), (h2, h1), (h1, h2)]
    layers = []
    for b in bits:
        ops = []
        for n, k in shapes:
            w = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
            ops.append(qweight.quantize(w, b))
            del w
        lns = [(torch.ones(h1, device=dev) if j % 2 == 0 else torch.zeros(h1, device=dev)).to(torch.bfloat16)
               for j in range(4)]
        layers.append((ops, lns))
    x0 = torch.randn(m, h1, device=dev).to(torch.bfloat16)
    x = x0.clone()
    plan = qweight.DecodePlan(layers, x)
    info = plan.info()

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        return sorted(ts)[len(ts) // 2]

    t_fused = timed(lambda: plan.run(torch.cuda.current_stream()))
    res = {"layers": len(bits), "h1": h1, "h2": h2, "m": m, "grid": info["grid"],
           "weight_MB": info["weight_bytes"] / 1e6, "fused_us": t_fused * 1e6,
           "fused_GBs": info["alg_bytes"] / t_fused / 1e9, "fused_us_per_layer": t_fused * 1e6 / len(bits)}
    if args.per_op:
        a = torch.empty(m, h1, dtype=torch.bfloat16, device=dev)
        qkv = torch.empty(m, 3 * h1, dtype=torch.bfloat16, device=dev)
        f = torch.empty(m, h2, dtype=torch.bfloat16, device=dev)
        xp = x0.clone()

        def per_op():
            for ops, ln in layers:
                check(lib.hp_layernorm(xp.data_ptr(), h1, m, h1, ln[0].data_ptr(), ln[1].data_ptr(),
                                       a.data_ptr(), h1, None))
                qweight.qlinear(ops[0], a, out=qkv)
                qweight.qlinear(ops[1], qkv[:, 2 * h1:], out=xp, residual=xp)
                check(lib.hp_layernorm(xp.data_ptr(), h1, m, h1, ln[2].data_ptr(), ln[3].data_ptr(),
                                       a.data_ptr(), h1, None))
                qweight.qlinear(ops[2], a, out=f, relu=True)
                qweight.qlinear(ops[3], f, out=xp, residual=xp)
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            per_op()
            st.synchronize()
            with torch.cuda.graph(g, stream=st):
                per_op()
        t_op = timed(lambda: g.replay())
        res.update({"per_op_graph_us": t_op * 1e6, "per_op_GBs": info["alg_bytes"] / t_op / 1e9})
    print(json.dumps(res), flush=True)
    plan.close()


if __name__ == "__main__":
    main()
