"""K3 fused decode step (hp_decode_plan_*): one persistent kernel per decode
step of a layer stack must be BIT-IDENTICAL to the per-op launches of the
same stack (hp_layernorm + hp_qlinear decode, the same stream-K
segmentation and reduction order), across mixed 3/4/8/16-bit layers, both
schemes, m in {1, 8, 32}, CUDA-graph replay, and repeated runs (the
in-kernel completion counters reset themselves)."""
import pytest

pytestmark = pytest.mark.gpu


def _stack(dev, bits, h1, h2, scheme, seed=0):
    import torch
    from paper_2403_01136_b200 import capi, qweight
    g = torch.Generator(device="cpu").manual_seed(seed)
    layers = []
    shapes = [(3 * h1, h1), (h1, h1), (h2, h1), (h1, h2)]
    for b in bits:
        ops = []
        for n, k in shapes:
            w = (torch.randn(n, k, generator=g) * 0.02).to(torch.bfloat16).to(dev)
            ops.append(qweight.quantize(w, b, scheme=scheme))
        lns = []
        for j in range(4):
            base = 1.0 if j % 2 == 0 else 0.0
            lns.append((base + 0.02 * torch.randn(h1, generator=g)).to(torch.bfloat16).to(dev))
        layers.append((ops, lns))
    return layers


def _per_op(layers, x, h1, h2):
    import torch
    from paper_2403_01136_b200 import qweight
    from paper_2403_01136_b200.capi import check, lib
    m = x.shape[0]
    a = torch.empty(m, h1, dtype=torch.bfloat16, device=x.device)
    qkv = torch.empty(m, 3 * h1, dtype=torch.bfloat16, device=x.device)
    f = torch.empty(m, h2, dtype=torch.bfloat16, device=x.device)
    for ops, ln in layers:
        check(lib.hp_layernorm(x.data_ptr(), h1, m, h1, ln[0].data_ptr(), ln[1].data_ptr(),
                               a.data_ptr(), h1, None))
        qweight.qlinear(ops[0], a, out=qkv)
        qweight.qlinear(ops[1], qkv[:, 2 * h1:], out=x, residual=x)
        check(lib.hp_layernorm(x.data_ptr(), h1, m, h1, ln[2].data_ptr(), ln[3].data_ptr(),
                               a.data_ptr(), h1, None))
        qweight.qlinear(ops[2], a, out=f, relu=True)
        qweight.qlinear(ops[3], f, out=x, residual=x)
    return x


@pytest.mark.parametrize("m", [1, 8, 32])
@pytest.mark.parametrize("scheme", [1, 0])
def test_fused_matches_per_op_bitwise(cuda, m, scheme):
    import torch
    from paper_2403_01136_b200 import qweight
    h1, h2 = 768, 3072
    layers = _stack(cuda, [3, 4, 8, 16, 4], h1, h2, scheme)
    x0 = torch.randn(m, h1, device=cuda).to(torch.bfloat16)
    ref = _per_op(layers, x0.clone(), h1, h2)
    x = x0.clone()
    plan = qweight.DecodePlan(layers, x)
    plan.run()
    torch.cuda.synchronize()
    assert torch.isfinite(x.float()).all()
    assert torch.equal(x, ref), float((x.float() - ref.float()).abs().max())
    # replay: counters reset in-kernel
    for _ in range(3):
        x.copy_(x0)
        plan.run()
    torch.cuda.synchronize()
    assert torch.equal(x, ref)
    plan.close()


def test_fused_opt13b_shapes_and_graph(cuda):
    import torch
    from paper_2403_01136_b200 import qweight
    h1, h2 = 5120, 20480
    layers = _stack(cuda, [16, 8, 4, 3], h1, h2, 1, seed=3)
    x0 = torch.randn(32, h1, device=cuda).to(torch.bfloat16)
    ref = _per_op(layers, x0.clone(), h1, h2)
    x = x0.clone()
    plan = qweight.DecodePlan(layers, x)
    torch.cuda.synchronize()  # ref/x come from the default stream
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        plan.run(st)
        st.synchronize()
        assert torch.equal(x, ref)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            plan.run(st)
    for _ in range(2):
        x.copy_(x0)
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(x, ref)
    info = plan.info()
    assert info["ops"] == 6 * 4 and info["weight_bytes"] > 0
    plan.close()
