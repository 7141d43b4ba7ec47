"""Determinism / parity diagnostic for prefill stream-K splits (one GPU)."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))


def main():
    from paper_2403_01136_b200 import qweight
    dev = torch.device("cuda:0")
    for (n, k, m) in ((5120, 512, 2048), (5120, 5120, 2048), (5120, 20480, 2048)):
        for bits in tuple(int(b) for b in os.environ.get("DIAG_BITS", "16,4").split(",")):
            g = torch.Generator().manual_seed(5)
            w = (torch.randn(n, k, generator=g) * 0.02).to(torch.bfloat16).to(dev)
            x = torch.randn(m, k, generator=g).to(torch.bfloat16).to(dev)
            qw = qweight.quantize(w, bits)
            for waves in (None, "0", "1"):
                if waves is None:
                    os.environ.pop("HP_PREFILL_DP_WAVES", None)
                else:
                    os.environ["HP_PREFILL_DP_WAVES"] = waves
                ys = [qweight.qlinear(qw, x, phase=0) for _ in range(6)]
                torch.cuda.synchronize()
                d = [float((y.float() - ys[0].float()).abs().max()) for y in ys[1:]]
                neq = [int((y != ys[0]).sum()) for y in ys[1:]]
                print(n, k, m, bits, waves, "maxdiff", d, "n_neq", neq, flush=True)


if __name__ == "__main__":
    main()
