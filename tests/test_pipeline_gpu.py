"""End-to-end serving round on one B200 through the C-ABI pipeline (OPT
decoder: token + position embedding, per layer LN -> qkv -> causal attention
over the KV cache -> out(+res) -> LN -> fc1(relu) -> fc2(+res), final LN,
tied LM head, greedy argmax).

Reference: a torch fp32 decoder built on ORACLE-dequantized weights
(oracle/hp_oracle.c quantize() restatement, zero + (code - off) * step,
indicator.cpp:53) of the same synthetic checkpoint (oracle/synth.py seeds),
rounding to bf16 wherever the runtime stores bf16. It is teacher-forced
with the runtime's generated tokens (one causal pass over prompt + tokens),
so a near-tie argmax flip cannot derail the comparison: every generated
token must be the reference's argmax up to a logit margin, and the final
hidden state of the last position must match within the tolerance.
Plan: the OPT-125M fixture from the reference planner
(tests/golden/plans/opt125m_b8_1gpu.json), B=8, s=512.
"""
import json

import numpy as np
import pytest

from tests.util import bits_to_torch

pytestmark = pytest.mark.gpu

H1, H2, HEADS, VOCAB, POS = 768, 3072, 12, 50272, 2050
SHAPES = [(3 * H1, H1), (H1, H1), (H2, H1), (H1, H2)]


def _plan(n=4, eta=None, xi=None):
    from paper_2403_01136_b200.pipeline import load_plan
    plan_json, model_json = load_plan("opt125m_b8_1gpu")
    plan = json.loads(plan_json)
    plan["workload"]["n"] = n  # xi == B: the objective does not depend on n
    if xi is not None:  # several decode groups (the last one ragged when B % xi != 0)
        plan["xi"] = xi
    if eta is not None or xi is not None:  # re-batch; recompose Eq. (4) (types.cpp:17-24)
        eta = plan["eta"] if eta is None else eta
        plan["eta"] = eta
        o, B = plan["objective"], plan["workload"]["global_bz"]
        bc = lambda u: -(-(B - u) // u)
        o["total"] = (bc(eta) * o["t_max_pre"] + bc(plan["xi"]) * (n - 1) * o["t_max_dec"]
                      + o["t_pre_total"] + o["t_dec_total"] + o["theta"] * o["omega_sum"])
    return plan, model_json


def _synth(n, seed, mean, std):
    from oracle import synth
    return synth.synth_bits(n, seed, mean, std)


def _checkpoint(bits):
    """bf16 bit patterns of every tensor of the synthetic checkpoint."""
    from oracle import synth
    ck = {"linear": [], "norm": []}
    for i in range(len(bits)):
        for o, (nn, kk) in enumerate(SHAPES):
            ck["linear"].append(_synth(nn * kk, synth.seed_for(1, i, o), 0.0, 0.02).reshape(nn, kk))
        for j in range(4):
            ck["norm"].append(_synth(H1, synth.seed_for(4, i, j), 1.0 if j % 2 == 0 else 0.0, 0.02))
    ck["embed"] = _synth(VOCAB * H1, synth.seed_for(6), 0.0, 0.02).reshape(VOCAB, H1)
    ck["pos"] = _synth(POS * H1, synth.seed_for(7), 0.0, 0.02).reshape(POS, H1)
    ck["lnf"] = [_synth(H1, synth.seed_for(8, j), 1.0 if j == 0 else 0.0, 0.02) for j in range(2)]
    return ck


def _ref_logits_and_hidden(plan, ck, tokens, dev):
    """Teacher-forced reference over prompt + generated tokens [B, s + n - 1]."""
    import torch

    import oracle
    port = oracle.port()
    ws = []
    for i, b in enumerate(plan["layer_bits"]):
        lw = []
        for o in range(4):
            wb = ck["linear"][4 * i + o]
            if b == 16:
                lw.append(bits_to_torch(wb, dev).float())
            else:
                codes, step, zero = port.quantize_matrix(wb, b, 1)
                off = (1 << (b - 1)) - 1
                k = wb.shape[1]
                w = zero.repeat(128, axis=1)[:, :k] + (codes.astype(np.float64) - off) * step.repeat(128, axis=1)[:, :k]
                lw.append(torch.from_numpy(w).to(dev).float())
        ln = [bits_to_torch(ck["norm"][4 * i + j], dev).float() for j in range(4)]
        ws.append((lw, ln))
    E = bits_to_torch(ck["embed"], dev).float()
    P = bits_to_torch(ck["pos"], dev).float()
    lnf = [bits_to_torch(v, dev).float() for v in ck["lnf"]]

    def bf(t):
        return t.to(torch.bfloat16).float()

    def ln_(x, g, b):
        mu = x.mean(-1, keepdim=True)
        var = ((x - mu) ** 2).mean(-1, keepdim=True)
        return bf((x - mu) * torch.rsqrt(var + 1e-5) * g + b)

    tok = torch.from_numpy(tokens).to(dev).long()
    B, T = tok.shape
    x = bf(E[tok] + P[torch.arange(T, device=dev) + 2])
    mask = torch.ones(T, T, dtype=torch.bool, device=dev).tril()
    for lw, ln in ws:
        a = ln_(x, ln[0], ln[1])
        qkv = bf(a @ lw[0].T)
        q, k, v = (qkv[..., j * H1:(j + 1) * H1].reshape(B, T, HEADS, H1 // HEADS) for j in range(3))
        sc = torch.einsum("bthd,bshd->bhts", q, k) / np.sqrt(H1 // HEADS)
        sc = sc.masked_fill(~mask, float("-inf"))
        att = bf(torch.einsum("bhts,bshd->bthd", torch.softmax(sc, -1), v).reshape(B, T, H1))
        x = bf(x + att @ lw[1].T)
        a = ln_(x, ln[2], ln[3])
        f = bf(torch.relu(a @ lw[2].T))
        x = bf(x + f @ lw[3].T)
    logits = bf(ln_(x, lnf[0], lnf[1]) @ E.T)
    return logits, x


def _run(pipe, B, n, host_tokens=None):
    import torch
    out = torch.empty(B * n, dtype=torch.int32).pin_memory()
    pipe.run(host_tokens.data_ptr() if host_tokens is not None else None, out.data_ptr())
    return out.clone()


def _final_hidden(pipe, B):
    import torch
    h = torch.empty(B * H1, dtype=torch.bfloat16)
    pipe.final_hidden(h.data_ptr())
    return h.reshape(B, H1)


@pytest.mark.parametrize("graphs,eta,xi", [(True, None, None), (False, None, None), (True, 3, None),
                                           (True, None, 3)])
def test_opt125m_round_matches_reference_decoder(cuda, graphs, eta, xi):
    """eta = 3 with B = 8: a ragged last prefill micro-batch (3, 3, 2), the
    case whose stream-K workspace was once undersized. xi = 3:
    three decode groups (3, 3, 2) interleaved by the schedule, the last one
    ragged -- different K3 tile widths and KV-cache request offsets per group."""
    import torch

    from oracle import synth
    from paper_2403_01136_b200.pipeline import Pipeline
    n = 4
    plan, model_json = _plan(n, eta, xi)
    B, s = 8, 512
    pipe = Pipeline(json.dumps(plan), model_json, use_graphs=graphs, instrument=True)
    gen = _run(pipe, B, n)
    gen2 = _run(pipe, B, n)  # graph replay path when graphs=True
    assert torch.equal(gen, gen2)
    hid = _final_hidden(pipe, B).float()
    ks = [pipe.kernel_stats(k) for k in range(4)]
    pipe.close()
    assert all(k["launches"] > 0 and k["seconds"] > 0 for k in ks)
    gen = gen.reshape(B, n).numpy()
    prompt = synth.synth_tokens(B * s, synth.seed_for(3), VOCAB).reshape(B, s)
    assert ((gen >= 0) & (gen < VOCAB)).all()
    ck = _checkpoint(plan["layer_bits"])
    seq = np.concatenate([prompt, gen[:, :n - 1]], axis=1)  # positions 0 .. s + n - 2
    logits, x = _ref_logits_and_hidden(plan, ck, seq, cuda)
    lg = logits[:, s - 1:].cpu()  # the logits that chose tokens 0 .. n-1
    top = lg.max(dim=-1).values
    picked = lg.gather(-1, torch.from_numpy(gen).long()[..., None])[..., 0]
    # every generated token is the reference argmax up to a small logit margin
    margin = float((top - picked).max())
    assert margin < 0.05, margin
    agree = float((lg.argmax(-1).numpy() == gen).mean())
    assert agree >= 0.9, agree
    ref = x[:, -1].cpu()
    err = float((hid - ref).abs().max() / ref.abs().max())
    assert err < 2e-2, err


def test_graph_and_eager_bit_identical(cuda):
    import torch
    from paper_2403_01136_b200.pipeline import Pipeline
    plan, model_json = _plan(3)
    outs, hids = [], []
    for graphs in (True, False):
        pipe = Pipeline(json.dumps(plan), model_json, use_graphs=graphs)
        _run(pipe, 8, 3)
        outs.append(_run(pipe, 8, 3))
        hids.append(_final_hidden(pipe, 8))
        pipe.close()
    assert torch.equal(outs[0], outs[1]) and torch.equal(hids[0], hids[1])


def test_host_prompt_tokens_path(cuda):
    """e2e path: the prompt token ids come from pinned host memory."""
    import torch

    from oracle import synth
    from paper_2403_01136_b200.pipeline import Pipeline
    plan, model_json = _plan(2)
    pipe = Pipeline(json.dumps(plan), model_json)
    host = torch.from_numpy(synth.synth_tokens(8 * 512, synth.seed_for(3), VOCAB)).pin_memory()
    a = _run(pipe, 8, 2)
    b = _run(pipe, 8, 2, host)
    assert torch.equal(a, b)  # same ids whether resident or uploaded
    other = host.clone()
    other[:512] = 7  # request 0 gets a different prompt
    c = _run(pipe, 8, 2, other.pin_memory())
    assert torch.equal(c.reshape(8, 2)[1:], a.reshape(8, 2)[1:])  # requests are independent
    pipe.close()


def _weight_set(ck, plan, mode, tmp_path=None, bin_bytes=1 << 20):
    """The synthetic checkpoint handed over explicitly: pageable numpy
    buffers, pinned torch tensors, or one raw bf16 file with offsets."""
    import torch
    from paper_2403_01136_b200.pipeline import WeightSet
    L = len(plan["layer_bits"])
    w = WeightSet(L, bin_bytes=bin_bytes)
    tensors = ([("linear", i, a) for i, a in enumerate(ck["linear"])] +
               [("norm", i, a) for i, a in enumerate(ck["norm"])] +
               [("embed", 0, ck["embed"]), ("pos", 0, ck["pos"]),
                ("final_norm", 0, ck["lnf"][0]), ("final_norm", 1, ck["lnf"][1])])
    if mode == "file":
        path = tmp_path / "ckpt.bf16"
        off = 0
        with open(path, "wb") as f:
            for kind, i, a in tensors:
                buf = np.ascontiguousarray(a).tobytes()
                f.write(buf)
                _assign(w, kind, i, (path, off))
                off += len(buf)
        return w
    for kind, i, a in tensors:
        a = np.ascontiguousarray(a)
        if mode == "pinned":
            a = torch.from_numpy(a.view(np.int16)).pin_memory()
        _assign(w, kind, i, a)
    return w


def _assign(w, kind, i, v):
    if kind in ("linear", "norm"):
        getattr(w, kind)[i] = v
    elif kind == "final_norm":
        w.final_norm[i] = v
    else:
        setattr(w, kind, v)


@pytest.mark.parametrize("mode", ["pageable", "pinned", "file"])
def test_weight_loader_bit_identical_to_synthetic(cuda, tmp_path, mode):
    """The binned host/disk -> device loader with K1 per bin (1 MiB bins:
    several 128-row blocks per op) serves exactly the weights the device
    generator makes: generated tokens and final hidden states bit-identical."""
    import torch
    from paper_2403_01136_b200.pipeline import Pipeline
    plan, model_json = _plan(3)
    base = Pipeline(json.dumps(plan), model_json)
    ref_tok, ref_hid = _run(base, 8, 3), _final_hidden(base, 8)
    base.close()
    ck = _checkpoint(plan["layer_bits"])
    ws = _weight_set(ck, plan, mode, tmp_path)
    pipe = Pipeline(json.dumps(plan), model_json, weights=ws)
    st = pipe.load_stats()
    tok, hid = _run(pipe, 8, 3), _final_hidden(pipe, 8)
    pipe.close()
    assert torch.equal(tok, ref_tok) and torch.equal(hid, ref_hid)
    src = sum(a.size for a in ck["linear"] + ck["norm"] + ck["lnf"]) * 2 + (ck["embed"].size + ck["pos"].size) * 2
    assert st["source_bytes"] == src
    assert st["bins"] > 4 * 12 and st["seconds"] > 0


def test_weight_loader_rejects_bad_sources(cuda, tmp_path):
    from paper_2403_01136_b200 import capi
    from paper_2403_01136_b200.pipeline import Pipeline, WeightSet
    plan, model_json = _plan(2)
    w = WeightSet(12)
    w.linear[0] = (tmp_path / "missing.bf16", 0)
    with pytest.raises(capi.InvalidArgument):
        Pipeline(json.dumps(plan), model_json, weights=w)
    short = tmp_path / "short.bf16"
    short.write_bytes(b"\0" * 1000)
    w = WeightSet(12)
    w.linear[1] = (short, 0)
    with pytest.raises(capi.InvalidArgument):
        Pipeline(json.dumps(plan), model_json, weights=w)
