"""Debug helper: K1 codes vs the golden matrix, per (bits, scheme), with the first mismatches."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from tests.util import bits_to_torch, bf16_bits_to_f64  # noqa: E402


def main():
    import torch
    from paper_2403_01136_b200 import qweight
    g = np.load(ROOT / "tests" / "golden" / "quant_golden.npz")
    for tag in ("aligned", "ragged"):
        wb = g[f"mat/{tag}/w_bits"]
        w64 = bf16_bits_to_f64(wb)
        for bits in (3, 4, 8):
            for scheme in (0, 1):
                key = f"mat/{tag}/b{bits}s{scheme}"
                qw, step64, zero64 = qweight.quantize(bits_to_torch(wb, "cuda"), bits, scheme, want_fp64=True)
                codes, _, _ = qweight.unpack(qw)
                c = codes.cpu().numpy()
                want = g[key + "/codes"]
                bad = np.argwhere(c != want)
                st_bad = int((step64.cpu().numpy().view(np.uint64) != g[key + "/step"].view(np.uint64)).sum())
                print(tag, bits, scheme, "code mismatches", len(bad), "of", c.size, "step mismatches", st_bad)
                for r, k in bad[:4]:
                    s = g[key + "/step"][r, k // 128]
                    z = g[key + "/zero"][r, k // 128]
                    print("   ", r, k, "w", w64[r, k], "got", c[r, k], "want", want[r, k], "X", (w64[r, k] - z) / s if s else None)


if __name__ == "__main__":
    main()
