"""Back-to-back qlinear launches inside a CUDA graph (no host gaps), cycling
through enough distinct weight copies that the working set (>= 1 GB) is far
larger than L2 — per-launch GPU time with weights streamed from HBM."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2403_01136_b200 import qweight
    dev = torch.device("cuda:0")
    shapes = [(20480, 5120, 4), (5120, 5120, 4), (15360, 5120, 16), (5120, 20480, 3),
              (15360, 5120, 3), (28672, 7168, 4), (7168, 28672, 8)]
    if len(sys.argv) > 1:
        shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
    for (n, k, bits) in shapes:
        w = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
        q0 = qweight.quantize(w, bits)
        copies = max(2, int((1 << 30) // q0.nbytes) + 1)
        qws = [q0] + [qweight.quantize(w, bits) for _ in range(copies - 1)]
        del w
        x = torch.randn(32, k, device=dev).to(torch.bfloat16)
        y = torch.empty(32, n, dtype=torch.bfloat16, device=dev)
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            for q in qws[:2]:
                qweight.qlinear(q, x, phase=1, out=y)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for q in qws:
                    qweight.qlinear(q, x, phase=1, out=y)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e3 / (3 * len(qws))
        wb = q0.nbytes + 2 * 32 * (n + k)
        print(f"{n}x{k} b{bits}: {t:.1f} us/launch ({wb / t / 1e3:.0f} GB/s, "
              f"{wb / t / 1e3 / 6545.6:.1%} of HBM) [{len(qws)} weight copies]", flush=True)
        del qws


if __name__ == "__main__":
    main()
