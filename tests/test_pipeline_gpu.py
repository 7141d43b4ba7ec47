"""End-to-end stage execution on one B200 through the C-ABI pipeline.

The runtime generates its own synthetic weights on the device (mirror of
oracle/synth.py) and quantizes them with K1; the test rebuilds the same
layers from oracle/synth.py bits, dequantizes them with the SAME K1 codes
(hp_quant_pack + hp_dequant) and runs a torch reference forward that rounds
to bf16 where the runtime stores bf16, so the comparison isolates the
GEMM accumulation order. Plan: the OPT-125M fixture from the reference
planner (tests/golden/plans/opt125m_b8_1gpu.json), B=8, s=512.
"""
import json

import numpy as np
import pytest

from tests.util import bits_to_torch

pytestmark = pytest.mark.gpu

H1, H2 = 768, 3072


def _plan(n=4):
    from paper_2403_01136_b200.pipeline import load_plan
    plan_json, model_json = load_plan("opt125m_b8_1gpu")
    plan = json.loads(plan_json)
    plan["workload"]["n"] = n  # xi == B: the objective does not depend on n
    return plan, model_json


def _ref_forward(plan, dev, n):
    import torch
    from oracle import synth
    from paper_2403_01136_b200 import qweight
    shapes = [(3 * H1, H1), (H1, H1), (H2, H1), (H1, H2)]
    layers = []
    for i, b in enumerate(plan["layer_bits"]):
        ws = []
        for o, (nn, kk) in enumerate(shapes):
            wb = synth.synth_bits(nn * kk, synth.seed_for(1, i, o), 0.0, 0.02).reshape(nn, kk)
            w = bits_to_torch(wb, dev)
            ws.append(qweight.dequant(qweight.quantize(w, b)).float() if b != 16 else w.float())
        ln = [bits_to_torch(synth.synth_bits(H1, synth.seed_for(4, i, j), 1.0 if j % 2 == 0 else 0.0,
                                             0.02), dev).float() for j in range(4)]
        layers.append((ws, ln))
    B, s = plan["workload"]["global_bz"], plan["workload"]["s"]
    x = bits_to_torch(synth.synth_bits(B * s * H1, synth.seed_for(3), 0.0, 1.0), dev).reshape(B * s, H1)

    def bf(t):
        return t.to(torch.bfloat16).float()

    def ln_(x, g, b):
        mu = x.mean(-1, keepdim=True)
        var = ((x - mu) ** 2).mean(-1, keepdim=True)
        return bf((x - mu) * torch.rsqrt(var + 1e-5) * g + b)

    def stack(x):
        x = x.float()
        for ws, ln in layers:
            a = ln_(x, ln[0], ln[1])
            qkv = bf(a @ ws[0].T)
            x = bf(qkv[:, 2 * H1:] @ ws[1].T + x)
            a = ln_(x, ln[2], ln[3])
            f = bf(torch.relu(a @ ws[2].T))
            x = bf(f @ ws[3].T + x)
        return x

    eta = plan["eta"]
    outs = []
    for k in range(0, B, eta):
        y = stack(x[k * s:(k + eta) * s])
        outs.append(y.reshape(-1, s, H1)[:, -1])
    d = torch.cat(outs)
    for _ in range(n - 1):
        d = stack(d)
    return d


@pytest.mark.parametrize("graphs", [True, False])
def test_opt125m_stage_matches_reference(cuda, graphs):
    import torch
    from paper_2403_01136_b200.pipeline import Pipeline
    n = 4
    plan, model_json = _plan(n)
    pipe = Pipeline(json.dumps(plan), model_json, use_graphs=graphs, instrument=True)
    out = torch.empty(8 * H1, dtype=torch.bfloat16).pin_memory()
    t = pipe.run(None, out.data_ptr())
    t2 = pipe.run(None, out.data_ptr())  # graph replay path when graphs=True
    assert t.makespan_s > 0 and t2.makespan_s > 0
    got = out.float().reshape(8, H1)
    ref = _ref_forward(plan, cuda, n).cpu()
    assert torch.isfinite(got).all()
    err = float((got - ref).abs().max() / ref.abs().max())
    assert err < 2e-2, err
    ks = pipe.kernel_stats(1)
    assert ks["launches"] > 0 and ks["seconds"] > 0
    pipe.close()


def test_graph_and_eager_bit_identical(cuda):
    import torch
    from paper_2403_01136_b200.pipeline import Pipeline
    plan, model_json = _plan(3)
    outs = []
    for graphs in (True, False):
        pipe = Pipeline(json.dumps(plan), model_json, use_graphs=graphs)
        o = torch.empty(8 * H1, dtype=torch.bfloat16).pin_memory()
        pipe.run(None, o.data_ptr())
        pipe.run(None, o.data_ptr())
        outs.append(o.clone())
        pipe.close()
    assert torch.equal(outs[0], outs[1])


def test_host_prompt_path(cuda):
    """e2e path: the prompt comes from pinned host memory."""
    import torch
    from oracle import synth
    from paper_2403_01136_b200.pipeline import Pipeline
    plan, model_json = _plan(2)
    pipe = Pipeline(json.dumps(plan), model_json)
    host_in = torch.from_numpy(synth.synth_bits(8 * 512 * H1, synth.seed_for(3), 0.0, 1.0)
                               .view(np.int16)).view(torch.bfloat16).pin_memory()
    a = torch.empty(8 * H1, dtype=torch.bfloat16).pin_memory()
    b = torch.empty(8 * H1, dtype=torch.bfloat16).pin_memory()
    pipe.run(None, a.data_ptr())
    pipe.run(host_in.data_ptr(), b.data_ptr())
    assert torch.equal(a, b)  # same bits whether the prompt was resident or uploaded
    pipe.close()


def test_fused_decode_bit_identical_to_per_op(cuda):
    """K3 fused decode units (decode_fused: one persistent launch per
    bit-width run of the stage) produce the same bits as the default per-op
    K3 launches; the mixed 4/8 plan makes the stage several runs."""
    import torch
    from paper_2403_01136_b200.pipeline import Pipeline
    plan, model_json = _plan(5)
    outs, launches = [], []
    for fused in (True, False):
        pipe = Pipeline(json.dumps(plan), model_json, decode_fused=fused, instrument=True)
        o = torch.empty(8 * H1, dtype=torch.bfloat16).pin_memory()
        pipe.run(None, o.data_ptr())
        pipe.run(None, o.data_ptr())
        outs.append(o.clone())
        launches.append(pipe.info()["launches_per_round"])
        pipe.close()
    assert torch.equal(outs[0], outs[1])
    assert launches[0] < launches[1]
