"""Back-to-back qlinear launches inside a CUDA graph (no host gaps):
per-launch GPU time, alone and interleaved with a small torch kernel."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2403_01136_b200 import qweight
    dev = torch.device("cuda:0")
    N = 20
    for (n, k, bits) in ((20480, 5120, 4), (5120, 5120, 4), (15360, 5120, 16), (5120, 20480, 3)):
        w = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
        qw = qweight.quantize(w, bits)
        x = torch.randn(32, k, device=dev).to(torch.bfloat16)
        y = torch.empty(32, n, dtype=torch.bfloat16, device=dev)
        small = torch.zeros(1024, device=dev)
        qweight.qlinear(qw, x, phase=1, out=y)
        torch.cuda.synchronize()
        res = {}
        for mode in ("b2b", "interleaved"):
            s = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                qweight.qlinear(qw, x, phase=1, out=y)  # warm on this stream
                torch.cuda.synchronize()
                with torch.cuda.graph(g, stream=s):
                    for _ in range(N):
                        qweight.qlinear(qw, x, phase=1, out=y)
                        if mode == "interleaved":
                            small.add_(1.0)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            res[mode] = e0.elapsed_time(e1) * 1e3 / (5 * N)
        wb = qw.nbytes + 2 * 32 * (n + k)
        print(f"{n}x{k} b{bits}: b2b {res['b2b']:.1f} us ({wb / res['b2b'] / 1e3:.0f} GB/s), "
              f"interleaved {res['interleaved']:.1f} us", flush=True)


if __name__ == "__main__":
    main()
