"""B200 profiler -> latency model: time one decoder layer
(LN1, qkv, out(+res), LN2, fc1(relu), fc2(+res); the executor's layer) per
bit width on this GPU at the workload grid the reference's latency model is
fitted on (latcost.hpp: prefill (v, s), decode (v, s, t)), write the profile
CSV `device,bit,phase,v,s,t,latency_s`, and fit it with the build's
hetplan::latcost (hp_host_latency_fit) into the model JSON the reference
planner reads (serialize_model format).

  python tools/latency_profile.py [--h1 5120 --h2 20480] [--out tests/golden/plans/b200_opt13b]

Layer latency is CUDA-event timed over a CUDA-graph replay of `reps`
layers (distinct weights, >> L2), so it is the per-layer cost inside a
stage, not a cold single launch. The executor's layer has self-only
attention, so decode latency carries no (t + s) term beyond noise.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from paper_2403_01136_b200 import capi, qweight
    from paper_2403_01136_b200.capi import check, lib
    ap = argparse.ArgumentParser()
    ap.add_argument("--h1", type=int, default=5120)
    ap.add_argument("--h2", type=int, default=20480)
    ap.add_argument("--bits", default="3,4,8,16")
    ap.add_argument("--layers", type=int, default=6, help="distinct layers per timed graph")
    ap.add_argument("--device-name", default="b200")
    ap.add_argument("--out", default=str(ROOT / "tests" / "golden" / "plans" / "b200_opt13b"))
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    h1, h2 = args.h1, args.h2
    shapes = [(3 * h1, h1), (h1, h1), (h2, h1), (h1, h2)]
    pre_grid = [(v, s) for v in (1, 2, 4) for s in (128, 256, 512)]
    dec_grid = [(v, s, t) for v in (1, 8, 16, 32) for s in (128, 512) for t in (1, 50)]
    rows = []
    for bits in map(int, args.bits.split(",")):
        layers = []
        for _ in range(args.layers):
            ops = [qweight.quantize((torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16), bits)
                   for n, k in shapes]
            ln = [(torch.ones(h1, device=dev) if j % 2 == 0 else torch.zeros(h1, device=dev)).to(torch.bfloat16)
                  for j in range(4)]
            layers.append((ops, ln))
        mmax = max(v * s for v, s in pre_grid)
        x = torch.randn(mmax, h1, device=dev).to(torch.bfloat16)
        a = torch.empty(mmax, h1, dtype=torch.bfloat16, device=dev)
        qkv = torch.empty(mmax, 3 * h1, dtype=torch.bfloat16, device=dev)
        f = torch.empty(mmax, h2, dtype=torch.bfloat16, device=dev)

        def stack(m, phase):
            for ops, ln in layers:
                check(lib.hp_layernorm(x.data_ptr(), h1, m, h1, ln[0].data_ptr(), ln[1].data_ptr(),
                                       a.data_ptr(), h1, torch.cuda.current_stream().cuda_stream))
                qweight.qlinear(ops[0], a[:m], phase=phase, out=qkv[:m])
                qweight.qlinear(ops[1], qkv[:m, 2 * h1:], phase=phase, out=x[:m], residual=x[:m])
                check(lib.hp_layernorm(x.data_ptr(), h1, m, h1, ln[2].data_ptr(), ln[3].data_ptr(),
                                       a.data_ptr(), h1, torch.cuda.current_stream().cuda_stream))
                qweight.qlinear(ops[2], a[:m], phase=phase, out=f[:m], relu=True)
                qweight.qlinear(ops[3], f[:m], phase=phase, out=x[:m], residual=x[:m])

        def layer_time(m, phase):
            st = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(st):
                stack(m, phase)
                st.synchronize()
                with torch.cuda.graph(g, stream=st):
                    stack(m, phase)
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e-3 / len(layers))
            return sorted(ts)[len(ts) // 2]

        for v, s in pre_grid:
            t = layer_time(v * s, capi.HP_PREFILL)
            rows.append(f"{args.device_name},{bits},prefill,{v},{s},0,{t!r}")
            print(rows[-1], flush=True)
        cache = {}
        for v, s, tt in dec_grid:  # decode cost does not depend on (s, t) here: time once per v
            if v not in cache:
                cache[v] = layer_time(v, capi.HP_DECODE)
            rows.append(f"{args.device_name},{bits},decode,{v},{s},{tt},{cache[v]!r}")
            print(rows[-1], flush=True)
        del layers
        torch.cuda.empty_cache()
    csv = "device,bit,phase,v,s,t,latency_s\n" + "\n".join(rows) + "\n"
    out = Path(args.out)
    out.with_suffix(".profile.csv").write_text(csv)
    buf = C.create_string_buffer(1 << 20)
    need = C.c_int64()
    check(lib.hp_host_latency_fit(csv.encode(), buf, len(buf), C.byref(need)))
    model = buf.value.decode()
    out.with_suffix(".latency_model.json").write_text(model)
    print(json.dumps({g["phase"] + str(g["bit"]): g["residuals"] for g in json.loads(model)["groups"]}))


if __name__ == "__main__":
    main()
