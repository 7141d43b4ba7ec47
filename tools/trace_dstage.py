"""Per-op timeline of one K3-fused decode step (HP_DSTAGE_TRACE build):
for each op, when its inputs became visible (first/last CTA), when the
epilogues finished it, and how far the weight stream ran ahead.

  HP_LIB_PATH=.../libhetplan_b200_dtrace.so python tools/trace_dstage.py [bits] [layers]
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch
    from paper_2403_01136_b200 import qweight
    from paper_2403_01136_b200.capi import lib
    bits = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    nl = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    h1, h2, m = 5120, 20480, 32
    dev = torch.device("cuda:0")
    shapes = [(3 * h1, h1), (h1, h1), (h2, h1), (h1, h2)]
    layers = []
    for _ in range(nl):
        ops = [qweight.quantize((torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16), bits)
               for n, k in shapes]
        lns = [(torch.ones(h1, device=dev) if j % 2 == 0 else torch.zeros(h1, device=dev)).to(torch.bfloat16)
               for j in range(4)]
        layers.append((ops, lns))
    x = torch.randn(m, h1, device=dev).to(torch.bfloat16)
    plan = qweight.DecodePlan(layers, x)
    for _ in range(3):
        plan.run()
    torch.cuda.synchronize()
    lib.hp_debug_dstage_trace.argtypes = [C.c_void_p, C.c_int]
    buf = np.zeros(148 * 256 * 8, dtype=np.uint64)
    lib.hp_debug_dstage_trace(buf.ctypes.data, buf.size)
    t = buf.reshape(148, 256, 8).astype(np.int64)
    nops = plan.info()["ops"]
    t = t[:, :nops]
    t0 = t[t > 0].min()
    names = ["LN1", "qkv", "out", "LN2", "fc1", "fc2"]
    print("op      in_first  in_last | epi_first epi_last | dq_last  prod_last  (us from start)")
    for o in range(nops):
        def col(ev):
            v = t[:, o, ev]
            v = v[v > 0]
            return ((v.min() - t0) / 1e3, (v.max() - t0) / 1e3) if v.size else (float("nan"),) * 2
        i0, i1 = col(0)
        e0, e1 = col(1)
        _, d1 = col(2)
        _, p1 = col(3)
        print(f"{o:2d} {names[o % 6]:4s} {i0:8.2f} {i1:8.2f} | {e0:8.2f} {e1:8.2f} | {d1:8.2f} {p1:8.2f}")
    print("first epilogue segment per op, median over CTAs (us after tfull): stored, ticket, done")
    for o in range(nops):
        v = t[:, o, 4:8].astype(np.float64)
        ok = v[:, 0] > 0
        if ok.sum() == 0:
            continue
        d = (v[ok] - v[ok][:, :1]) / 1e3
        d[v[ok] == 0] = np.nan
        print(f"  op {o}: tfull at {np.median((v[ok,0]-t0)/1e3):7.2f}  +stored {np.nanmedian(d[:,1]):5.2f}  "
              f"+ticket {np.nanmedian(d[:,2]):5.2f}  +done {np.nanmedian(d[:,3]):5.2f}  (max done {np.nanmax(d[:,3]):5.2f})")
    for o in (1, 4):
        e = (t[:, o, 1] - t0) / 1e3
        d = (t[:, o, 2] - t0) / 1e3
        order = np.argsort(e)
        print(f"op {o}: latest CTAs (cta, epi_done, dq_done):",
              [(int(c), round(float(e[c]), 1), round(float(d[c]), 1)) for c in order[-8:]])
        print(f"op {o}: earliest CTAs:", [(int(c), round(float(e[c]), 1), round(float(d[c]), 1)) for c in order[:5]])
        print(f"op {o}: epi_done by CTA:", " ".join(f"{v:.0f}" for v in e))


if __name__ == "__main__":
    main()


def detail(op_index=1):
    pass
