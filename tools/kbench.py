"""Kernel micro-benchmark: one qlinear op shape at a time, CUDA-event timed
(L2 flushed between launches), reporting GB/s (K3) and TFLOP/s (K4).

  python tools/kbench.py [--op decode|prefill|both] [--bits 4] [--reps 20]
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
    ap.add_argument("--op", default="both")
    ap.add_argument("--bits", default="3,4,8,16")
    ap.add_argument("--shapes", default="15360x5120,5120x5120,20480x5120,5120x20480")
    ap.add_argument("--m-dec", type=int, default=32)
    ap.add_argument("--m-pre", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--no-flush", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    # L2 flush by READING 256 MB (clean lines: no write-back traffic leaks
    # into the timed kernel, unlike a zero_() flush)
    flush = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    res = []
    for shape in args.shapes.split(","):
        n, k = map(int, shape.split("x"))
        w = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
        for bits in map(int, args.bits.split(",")):
            qw = qweight.quantize(w, bits)
            for phase, m in ((1, args.m_dec), (0, args.m_pre)):
                if args.op == "decode" and phase == 0 or args.op == "prefill" and phase == 1:
                    continue
                x = (torch.randn(m, k, device=dev)).to(torch.bfloat16)
                y = torch.empty(m, n, dtype=torch.bfloat16, device=dev)
                for _ in range(3):
                    qweight.qlinear(qw, x, phase=phase, out=y)
                ts = []
                for _ in range(args.reps):
                    if not args.no_flush:
                        flush.sum()
                    # keep the GPU busy while the host enqueues e0 / kernel / e1, so
                    # the events bracket the kernel and not the host launch latency
                    torch.cuda._sleep(200_000)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    qweight.qlinear(qw, x, phase=phase, out=y)
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e-3)
                t = sorted(ts)[len(ts) // 2]
                wbytes = qw.nbytes
                byts = wbytes + 2 * m * (n + k)
                flops = 2.0 * m * n * k
                r = {"n": n, "k": k, "bits": bits, "m": m, "phase": "decode" if phase else "prefill",
                     "us": t * 1e6, "GBs": byts / t / 1e9, "TFs": flops / t / 1e12}
                res.append(r)
                print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
