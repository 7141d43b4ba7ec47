"""Decoder glue kernels (csrc/decoder.cu) against plain
torch fp32 references: causal prefill attention writing the KV cache,
decode attention over the cache (memcost.cpp:38-42 sizes; head-major
layout [B][heads][S_max][hd]), token + position embedding (OPT, offset 2)
and greedy argmax."""
import math

import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _ref_attn(q, k, v, causal):
    """q [T, H, D], k/v [S, H, D] fp32 -> [T, H*D]; causal: query t sees keys <= t."""
    import torch
    T, H, D = q.shape
    sc = torch.einsum("thd,shd->hts", q, k) / math.sqrt(D)
    if causal:
        S = k.shape[0]
        mask = torch.ones(T, S, dtype=torch.bool, device=q.device).tril()
        sc = sc.masked_fill(~mask, float("-inf"))
    p = torch.softmax(sc, dim=-1)
    return torch.einsum("hts,shd->thd", p, v).reshape(T, H * D)


@pytest.mark.parametrize("hd,heads,s", [(64, 12, 512), (128, 4, 512), (128, 3, 200), (64, 2, 77)])
def test_prefill_attention_and_cache_write(cuda, hd, heads, s):
    import torch
    from paper_2403_01136_b200 import qweight
    g = torch.Generator(device=cuda).manual_seed(hd + s)
    h, reqs, B, S_max = heads * hd, 3, 5, s + 40
    qkv = torch.randn(reqs * s, 3 * h, generator=g, device=cuda).to(torch.bfloat16)
    kc = torch.zeros(B, heads, S_max, hd, dtype=torch.bfloat16, device=cuda)
    vc = torch.zeros_like(kc)
    req0 = 1
    out = qweight.attention_prefill(qkv, reqs, s, hd, kc, vc, req0, S_max)
    torch.cuda.synchronize()
    kc, vc = kc.transpose(1, 2).reshape(B, S_max, h), vc.transpose(1, 2).reshape(B, S_max, h)
    for r in range(reqs):
        rows = qkv[r * s:(r + 1) * s].float()
        q, k, v = (rows[:, i * h:(i + 1) * h].reshape(s, heads, hd) for i in range(3))
        ref = _ref_attn(q, k, v, causal=True)
        got = out[r * s:(r + 1) * s].float()
        err = float((got - ref).abs().max() / ref.abs().max())
        assert err < TOL, (r, err)
        # cache rows 0..s-1 of request req0 + r hold this request's k / v exactly
        assert torch.equal(kc[req0 + r, :s], qkv[r * s:(r + 1) * s, h:2 * h])
        assert torch.equal(vc[req0 + r, :s], qkv[r * s:(r + 1) * s, 2 * h:])
    assert torch.count_nonzero(kc[0]) == 0 and torch.count_nonzero(kc[req0:req0 + reqs, s:]) == 0


@pytest.mark.parametrize("split", [1, 2, 3])
@pytest.mark.parametrize("hd,heads,p", [(128, 40, 611), (64, 12, 512), (128, 2, 0), (64, 3, 33)])
def test_decode_attention_appends_and_attends(cuda, hd, heads, p, split):
    import torch
    from paper_2403_01136_b200 import qweight
    g = torch.Generator(device=cuda).manual_seed(hd * 7 + p)
    h, rows, B, S_max = heads * hd, 6, 9, 612
    kh = torch.randn(B, heads, S_max, hd, generator=g, device=cuda).to(torch.bfloat16)
    vh = torch.randn(B, heads, S_max, hd, generator=g, device=cuda).to(torch.bfloat16)
    qkv = torch.randn(rows, 3 * h, generator=g, device=cuda).to(torch.bfloat16)
    req0 = 2
    k_before = kh.transpose(1, 2).reshape(B, S_max, h).clone()
    out = qweight.attention_decode(qkv, hd, p, kh, vh, req0, S_max, split=split)
    torch.cuda.synchronize()
    if split > 1:  # deterministic merge of the splits: a rerun gives the same bits
        assert torch.equal(out, qweight.attention_decode(qkv, hd, p, kh, vh, req0, S_max, split=split))
    # [B][S_max][h] views of the head-major caches for the checks below
    kc, vc = kh.transpose(1, 2).reshape(B, S_max, h), vh.transpose(1, 2).reshape(B, S_max, h)
    for r in range(rows):
        assert torch.equal(kc[req0 + r, p], qkv[r, h:2 * h])
        assert torch.equal(vc[req0 + r, p], qkv[r, 2 * h:])
        q = qkv[r, :h].float().reshape(1, heads, hd)
        k = kc[req0 + r, :p + 1].float().reshape(p + 1, heads, hd)
        v = vc[req0 + r, :p + 1].float().reshape(p + 1, heads, hd)
        ref = _ref_attn(q, k, v, causal=False)[0]
        err = float((out[r].float() - ref).abs().max() / ref.abs().max())
        assert err < TOL, (r, err)
    # nothing else in the cache changed
    k_before[req0:req0 + rows, p] = kc[req0:req0 + rows, p]
    assert torch.equal(k_before, kc)


def test_embed_token_plus_position(cuda):
    import torch
    from paper_2403_01136_b200 import qweight
    g = torch.Generator(device=cuda).manual_seed(3)
    vocab, h, pos_s, s = 1000, 256, 300, 40
    E = torch.randn(vocab, h, generator=g, device=cuda).to(torch.bfloat16)
    P = torch.randn(pos_s, h, generator=g, device=cuda).to(torch.bfloat16)
    tok = torch.randint(0, vocab, (3 * s,), generator=g, device=cuda, dtype=torch.int32)
    x = qweight.embed(tok, E, P, 0, pos_per_req=True, s_tokens=s)
    pos = torch.arange(3 * s, device=cuda) % s + 2
    ref = (E[tok.long()].float() + P[pos].float()).to(torch.bfloat16)
    assert torch.equal(x, ref)
    x = qweight.embed(tok[:5], E, P, 123)  # decode: one position for all rows
    assert torch.equal(x, (E[tok[:5].long()].float() + P[125].float()).to(torch.bfloat16))
    x = qweight.embed(tok[:5], E, None, 123)  # no learned positions (ALiBi models)
    assert torch.equal(x, E[tok[:5].long()])


def test_argmax_lowest_index_on_ties(cuda):
    import torch
    from paper_2403_01136_b200 import qweight
    g = torch.Generator(device=cuda).manual_seed(9)
    logits = torch.randn(7, 50272, generator=g, device=cuda).to(torch.bfloat16)
    logits[3, 100] = logits[3, 40000] = 50.0
    logits[5, :] = 1.0
    tok = qweight.argmax(logits)
    ref = logits.float().argmax(dim=1).to(torch.int32)  # torch returns the first max
    assert torch.equal(tok, ref)
    assert int(tok[3]) == 100 and int(tok[5]) == 0
