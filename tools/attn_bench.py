"""Decode / prefill attention micro-benchmark (glue kernels, csrc/decoder.cu):
OPT-13B shapes (40 heads x 128), xi = 32 requests, context p + 1 keys;
CUDA-graph of 20 launches over distinct KV caches (>> L2), CUDA events.

  python tools/attn_bench.py [--p 560]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2403_01136_b200 import qweight
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, default=560)
    ap.add_argument("--heads", type=int, default=40)
    ap.add_argument("--rows", type=int, default=32)
    ap.add_argument("--split", type=int, default=2)
    ap.add_argument("--prefill", action="store_true", help="causal prefill attention: --reqs x --s tokens")
    ap.add_argument("--reqs", type=int, default=4)
    ap.add_argument("--s", type=int, default=512)
    args = ap.parse_args()
    if args.prefill:
        return prefill(args)
    dev = torch.device("cuda:0")
    hd, S = 128, 612
    h = args.heads * hd
    caches = [(torch.randn(args.rows, S, h, device=dev).to(torch.bfloat16),
               torch.randn(args.rows, S, h, device=dev).to(torch.bfloat16)) for _ in range(12)]
    qkv = torch.randn(args.rows, 3 * h, device=dev).to(torch.bfloat16)
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for kc, vc in caches:
            qweight.attention_decode(qkv, hd, args.p, kc, vc, 0, S, split=args.split, stream=st)
        st.synchronize()
        with torch.cuda.graph(g, stream=st):
            for kc, vc in caches:
                qweight.attention_decode(qkv, hd, args.p, kc, vc, 0, S, split=args.split, stream=st)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3 / len(caches))
    t = sorted(ts)[2]
    byts = 2.0 * 2 * args.rows * (args.p + 1) * h
    peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
    print(json.dumps({"p": args.p, "split": args.split, "us": t * 1e6, "GBs": byts / t / 1e9, "frac": byts / t / 1e9 / peaks["hbm_gbs"]}))


def prefill(args):
    import torch
    from paper_2403_01136_b200 import qweight
    dev = torch.device("cuda:0")
    hd = 128
    h = args.heads * hd
    S = args.s + 8
    qkvs = [torch.randn(args.reqs * args.s, 3 * h, device=dev).to(torch.bfloat16) for _ in range(6)]
    kc = torch.zeros(args.reqs, S, h, dtype=torch.bfloat16, device=dev)
    vc = torch.zeros_like(kc)
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        for q in qkvs:
            qweight.attention_prefill(q, args.reqs, args.s, hd, kc, vc, 0, S, stream=st)
        st.synchronize()
        with torch.cuda.graph(g, stream=st):
            for q in qkvs:
                qweight.attention_prefill(q, args.reqs, args.s, hd, kc, vc, 0, S, stream=st)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3 / len(qkvs))
    t = sorted(ts)[2]
    flops = 2.0 * args.s * args.s * h * args.reqs  # causal: QK^T and PV over s^2/2 pairs
    print(json.dumps({"prefill": True, "s": args.s, "reqs": args.reqs, "us": t * 1e6, "TFs": flops / t / 1e12}))


if __name__ == "__main__":
    main()
