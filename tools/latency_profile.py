"""B200 profiler -> latency model: time one decoder layer
of the executor (LN1, qkv, causal attention over the KV cache, out(+res),
LN2, fc1(relu), fc2(+res)) per bit width on this GPU over the workload grid
the reference's latency model is fitted on (latcost.cpp:60-67: prefill
features [1, v, s, v s, v s^2], decode [1, v, v (t+s), (t+s)]), write the
profile CSV `device,bit,phase,v,s,t,latency_s`, fit it with the build's
Eigen-free hetplan::latcost (hp_host_latency_fit) into the model JSON the
reference planner reads, and report the held-out prediction error of that
fit (the paper's "< 6%" claim): every grid point marked
`held` is left out of the fit and predicted.

  python tools/latency_profile.py --preset opt-30b --out tests/golden/plans/b200_opt30b

Layer latency is CUDA-event timed over a CUDA-graph replay of `layers`
distinct layers (weights >> L2), i.e. the per-layer cost inside a stage.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

PRESETS = {"opt-13b": (5120, 20480, 40), "opt-30b": (7168, 28672, 56),
           "opt-66b": (9216, 36864, 72), "bloom-176b": (14336, 57344, 112),
           "opt-125m": (768, 3072, 12)}


def main():
    import torch
    from paper_2403_01136_b200 import capi, qweight
    from paper_2403_01136_b200.capi import check, lib
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="opt-13b")
    ap.add_argument("--bits", default="3,4,8,16")
    ap.add_argument("--layers", type=int, default=4, help="distinct layers per timed graph")
    ap.add_argument("--device-name", default="b200")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    h1, h2, heads = PRESETS[args.preset]
    hd = h1 // heads
    out = Path(args.out or ROOT / "tests" / "golden" / "plans" / f"b200_{args.preset.replace('-', '')}")
    shapes = [(3 * h1, h1), (h1, h1), (h2, h1), (h1, h2)]
    # (v, s, held-out?) / (v, s, t, held-out?)
    pre_grid = [(v, s, False) for v in (1, 2, 4, 8) for s in (128, 256, 512)] + \
               [(3, 384, True), (6, 192, True), (2, 448, True)]
    dec_grid = [(v, s, t, False) for v in (1, 8, 16, 32) for s in (128, 512) for t in (1, 50, 100)] + \
               [(24, 384, 30, True), (12, 256, 80, True), (32, 448, 64, True)]
    S_max = 512 + 101
    vmax_dec = max(v for v, *_ in dec_grid)
    rows, held = [], []
    for bits in map(int, args.bits.split(",")):
        layers = []
        for _ in range(args.layers):
            ops = [qweight.quantize((torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16), bits)
                   for n, k in shapes]
            ln = [(torch.ones(h1, device=dev) if j % 2 == 0 else torch.zeros(h1, device=dev)).to(torch.bfloat16)
                  for j in range(4)]
            layers.append((ops, ln))
        mmax = max(v * s for v, s, _ in pre_grid)
        x = torch.randn(mmax, h1, device=dev).to(torch.bfloat16)
        a = torch.empty(mmax, h1, dtype=torch.bfloat16, device=dev)
        qkv = torch.randn(mmax, 3 * h1, device=dev).to(torch.bfloat16)
        f = torch.empty(mmax, h2, dtype=torch.bfloat16, device=dev)
        nreq = max(8, vmax_dec)
        kc = torch.randn(nreq, S_max, h1, device=dev).to(torch.bfloat16)
        vc = torch.randn(nreq, S_max, h1, device=dev).to(torch.bfloat16)
        stream = lambda: torch.cuda.current_stream().cuda_stream
        # the executor's decode attention split (pipeline.cpp: one CTA per
        # (request, head) unless the pairs would not fill ~8 CTAs per SM)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count

        def attn_split(v):
            pairs = v * heads
            return max(1, min(8, -(-8 * sms // pairs)))
        aws_n = max(int(lib.hp_attention_decode_workspace_bytes(vmax_dec, h1, hd, attn_split(v)))
                    for v in range(1, vmax_dec + 1))
        aws = torch.zeros(max(aws_n, 1), dtype=torch.uint8, device=dev)

        def stack(v, s, t, phase):
            m = v * s if phase == capi.HP_PREFILL else v
            for ops, ln in layers:
                check(lib.hp_layernorm(x.data_ptr(), h1, m, h1, ln[0].data_ptr(), ln[1].data_ptr(),
                                       a.data_ptr(), h1, stream()))
                qweight.qlinear(ops[0], a[:m], phase=phase, out=qkv[:m])
                if phase == capi.HP_PREFILL:
                    check(lib.hp_attention_prefill(qkv.data_ptr(), v, s, h1, hd, a.data_ptr(),
                                                   kc.data_ptr(), vc.data_ptr(), 0, S_max, stream()))
                else:
                    check(lib.hp_attention_decode(qkv.data_ptr(), v, h1, hd, s + t - 1, a.data_ptr(),
                                                  kc.data_ptr(), vc.data_ptr(), 0, S_max, attn_split(v),
                                                  aws.data_ptr(), aws_n, stream()))
                qweight.qlinear(ops[1], a[:m], phase=phase, out=x[:m], residual=x[:m])
                check(lib.hp_layernorm(x.data_ptr(), h1, m, h1, ln[2].data_ptr(), ln[3].data_ptr(),
                                       a.data_ptr(), h1, stream()))
                qweight.qlinear(ops[2], a[:m], phase=phase, out=f[:m], relu=True)
                qweight.qlinear(ops[3], f[:m], phase=phase, out=x[:m], residual=x[:m])

        def layer_time(v, s, t, phase):
            st = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(st):
                stack(v, s, t, phase)
                st.synchronize()
                with torch.cuda.graph(g, stream=st):
                    stack(v, s, t, phase)
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e-3 / len(layers))
            return sorted(ts)[len(ts) // 2]

        for v, s, h in pre_grid:
            t = layer_time(v, s, 0, capi.HP_PREFILL)
            row = f"{args.device_name},{bits},prefill,{v},{s},0,{t!r}"
            (held if h else rows).append(row)
            print(row, "(held out)" if h else "", flush=True)
        for v, s, tt, h in dec_grid:
            t = layer_time(v, s, tt, capi.HP_DECODE)
            row = f"{args.device_name},{bits},decode,{v},{s},{tt},{t!r}"
            (held if h else rows).append(row)
            print(row, "(held out)" if h else "", flush=True)
        del layers, kc, vc
        torch.cuda.empty_cache()
    head = "device,bit,phase,v,s,t,latency_s\n"
    csv = head + "\n".join(rows) + "\n"
    out.with_suffix(".profile.csv").write_text(csv)
    out.with_suffix(".heldout.csv").write_text(head + "\n".join(held) + "\n")
    buf = C.create_string_buffer(1 << 20)
    need = C.c_int64()
    check(lib.hp_host_latency_fit(csv.encode(), buf, len(buf), C.byref(need)))
    model = buf.value.decode()
    out.with_suffix(".latency_model.json").write_text(model)
    errs = []
    for r in held:
        d, b, ph, v, s, t, lat = r.split(",")
        pred = C.c_double()
        check(lib.hp_host_latency_predict(model.encode(), d.encode(), int(b), 0 if ph == "prefill" else 1,
                                          float(v), float(s), float(t), C.byref(pred)))
        errs.append({"bit": int(b), "phase": ph, "v": int(v), "s": int(s), "t": int(t),
                     "measured_s": float(lat), "predicted_s": pred.value,
                     "rel_err": abs(pred.value - float(lat)) / float(lat)})
    summary = {"preset": args.preset, "fit_points": len(rows), "held_out": len(errs),
               "mean_abs_rel_err": sum(e["rel_err"] for e in errs) / len(errs),
               "max_abs_rel_err": max(e["rel_err"] for e in errs), "points": errs}
    out.with_suffix(".heldout_error.json").write_text(json.dumps(summary, indent=1))
    print(json.dumps({k: v for k, v in summary.items() if k != "points"}))


if __name__ == "__main__":
    main()
