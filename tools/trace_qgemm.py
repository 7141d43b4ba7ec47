"""Per-role pipeline trace of CTA 0 of one decode qlinear (HP_QGEMM_TRACE)."""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ["HP_QGEMM_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch
    from paper_2403_01136_b200 import qweight
    from paper_2403_01136_b200.capi import lib
    lib.hp_debug_trace.argtypes = [C.c_void_p, C.c_int]
    pos = [v for v in sys.argv[1:] if not v.startswith("--")]
    n, k, bits, m = (int(v) for v in (pos + ["20480", "5120", "4", "32"][len(pos):])[:4])
    dev = torch.device("cuda:0")
    w = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
    qw = qweight.quantize(w, bits)
    x = torch.randn(m, k, device=dev).to(torch.bfloat16)
    for _ in range(3):
        qweight.qlinear(qw, x, phase=(0 if m > 64 else 1))
    torch.cuda.synchronize()
    buf = np.zeros(6 * 64 * 4 + 13 * 1024, dtype=np.uint64)
    lib.hp_debug_trace(buf.ctypes.data, buf.size)
    cyc = buf[6 * 64 * 4 + 2048:6 * 64 * 4 + 2048 + 148].astype(np.int64)
    cta = buf[6 * 64 * 4:6 * 64 * 4 + 2048].reshape(1024, 2).astype(np.int64)
    cta = cta[cta[:, 0] > 0]
    t0c = cta[:, 0].min()
    ent = (cta[:, 0] - t0c) / 1000
    ext = (cta[:, 1] - t0c) / 1000
    print(f"CTAs {len(cta)}: entry min/med/max {ent.min():.2f}/{np.median(ent):.2f}/{ent.max():.2f} us; "
          f"exit min/med/max {ext.min():.2f}/{np.median(ext):.2f}/{ext.max():.2f} us")
    print("  exit sorted (last 10):", np.round(np.sort(ext)[-10:], 2), " argmax", int(np.argmax(ext)))
    if "--all" in sys.argv:
        print("  exit by CTA:", " ".join(f"{v:.1f}" for v in ext))
    smid = buf[6 * 64 * 4 + 2048 + 1024:6 * 64 * 4 + 2048 + 1024 + 148].astype(np.int64)
    if "--all" in sys.argv:
        print("  smid by CTA:", " ".join(str(v) for v in smid))
    mend = buf[6 * 64 * 4 + 4096:6 * 64 * 4 + 4096 + len(cta)].astype(np.int64)
    if mend.min() > 0:
        me = (mend - t0c) / 1000
        print(f"  last MMA issued min/med/max {me.min():.2f}/{np.median(me):.2f}/{me.max():.2f} us; "
              f"exit - last MMA med/max {np.median(ext - me):.2f}/{(ext - me).max():.2f} us; "
              f"slowest-MMA CTAs {np.argsort(me)[-5:].tolist()} on SMs "
              f"{[int(smid[i]) for i in np.argsort(me)[-5:]]}")
        if "--all" in sys.argv:
            print("  last MMA by CTA:", " ".join(f"{v:.1f}" for v in me))
    B2 = 6 * 64 * 4 + 5 * 1024
    nc = len(cta)
    fin = [buf[B2 + k * 1024:B2 + k * 1024 + nc].astype(np.int64) for k in range(8)]
    if fin[0].max() > 0 and mend.min() > 0:
        tf = np.where(fin[0] > 0, (fin[0] - t0c) / 1000, np.nan)
        st_ = np.where(fin[1] > 0, (fin[1] - t0c) / 1000, np.nan)
        tk = np.where(fin[2] > 0, (fin[2] - t0c) / 1000, np.nan)
        kind = fin[3]
        print(f"  final segment: tfull - lastMMA med {np.nanmedian(tf - me):.2f}; store {np.nanmedian(st_ - tf):.2f}; "
              f"ticket {np.nanmedian(tk - st_):.2f}; exit - (ticket or store) med "
              f"{np.nanmedian(ext - np.where(np.isnan(tk), st_, tk)):.2f} us")
        split = kind > 0
        last = (kind % 100) >= 10
        print(f"  final segments split: {int(split.sum())}/{nc}, of which reduced here: {int((split & last).sum())}")
        slow = np.argsort(ext)[-6:]
        for i in slow:
            rel = [(fin[k][i] - t0c) / 1000 if fin[k][i] > 0 else float("nan") for k in (4, 5, 6, 7)]
            print(f"    slow CTA {i} sm {int(smid[i])}: lastMMA {me[i]:.2f} tfull {tf[i]:.2f} stored {st_[i]:.2f} "
                  f"ticket {tk[i]:.2f} exit {ext[i]:.2f} kind {int(kind[i])} | loop exits: epi {rel[0]:.2f} "
                  f"act {rel[1]:.2f} prod {rel[2]:.2f} dq {rel[3]:.2f}")
    span_ns = (cta[:148, 1] - cta[:148, 0]).astype(np.float64)
    print(f"  CTA cycles/ns (implied GHz): median {np.median(cyc / span_ns):.3f}, cycles median {np.median(cyc):.0f}")
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        qweight.qlinear(qw, x, phase=(0 if m > 64 else 1))
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            for _ in range(10):
                qweight.qlinear(qw, x, phase=(0 if m > 64 else 1))
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    print(f"  graph b2b per launch: {e0.elapsed_time(e1) * 100:.1f} us")
    t = buf[:6 * 64 * 4].reshape(6, 64, 4).astype(np.int64)
    t0 = t[t > 0].min()
    if "--roles" not in sys.argv:
        return
    names = ["producer (start, empty_ok, issued)", "mma (start, full_ok, afull_ok, committed)",
             "dequant w4 (start, full_ok, aempty_ok, arrived)", "epilogue seg (start, tfull_ok, stored, fixup_done) @48..",
             "dequant w4 detail (codes_loaded, st_issued, st_done, -)",
             "fixup by segment (fence1_done, ticket, fence2_done[last], reduced[last])"]
    for r in range(6):
        print(names[r])
        for it in range(0, 64):
            row = t[r, it]
            if row.max() == 0:
                continue
            print(f"  it={it:2d} " + " ".join(f"{(v - t0) / 1000:8.2f}" if v else "       -" for v in row))


if __name__ == "__main__":
    main()
