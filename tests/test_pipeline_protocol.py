"""Multi-process check of the pipeline runtime's message protocol on CPU
(gloo, world size 2 and 4): every rank executes its static unit order
(hp_host_unit_order = pipesim::simulate order, as the C++ executor does),
receiving in the sender's order and sending after each unit exactly like
csrc/host/pipeline.cpp (stage r -> r+1 activations; last -> 0 feedback for
the next decode token). The run must complete (no deadlock) and every
message must carry the unit the receiver expects (no mismatch)."""
import ctypes as C
import json
import os
import socket
from pathlib import Path

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

PLANS = Path(__file__).resolve().parent / "golden" / "plans"


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _order(plan_json, model_json, stage):
    from paper_2403_01136_b200 import capi
    buf = (C.c_int * (3 * 100000))()
    n = C.c_int()
    capi.check(capi.lib.hp_host_unit_order(plan_json.encode(), model_json.encode(), stage, buf,
                                           100000, C.byref(n)))
    return [tuple(buf[3 * i:3 * i + 3]) for i in range(n.value)]


def _feedback_order(last_units, sched_groups, group_of_prefill, n):
    left = {}
    for g in group_of_prefill:
        left[g] = left.get(g, 0) + 1
    out = []
    for kind, idx, tok in last_units:
        if kind == 0:
            g = group_of_prefill[idx]
            left[g] -= 1
            if left[g] == 0 and n >= 2:
                out.append((1, g, 1))
        elif tok + 1 <= n - 1:
            out.append((1, idx, tok + 1))
    return out


def _worker(rank, world, port, plan_json, model_json, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = json.loads(plan_json)
    B, eta, xi, n = plan["workload"]["global_bz"], plan["eta"], plan["xi"], plan["workload"]["n"]
    group_of_prefill = [(k * eta) // xi for k in range(-(-B // eta))]
    orders = [_order(plan_json, model_json, j) for j in range(world)]
    mine = orders[rank]
    incoming = orders[rank - 1] if rank > 0 else _feedback_order(orders[-1], None, group_of_prefill, n)
    src = (rank - 1) % world
    dst = (rank + 1) % world
    inbox, got = {}, 0
    pending = []
    left = {}
    for g in group_of_prefill:
        left[g] = left.get(g, 0) + 1

    def tag(u):
        return torch.tensor(list(u), dtype=torch.int64)

    def recv_for(u):
        nonlocal got
        while u not in inbox:
            t = torch.zeros(3, dtype=torch.int64)
            dist.recv(t, src=src)
            exp = incoming[got]
            got += 1
            assert tuple(t.tolist()) == exp, (rank, tuple(t.tolist()), exp)
            inbox[exp] = True
        del inbox[u]

    last = rank == world - 1
    for u in mine:
        kind, idx, tok = u
        if rank > 0 or kind == 1:
            recv_for(u)
        if not last:
            pending.append(dist.isend(tag(u), dst=dst))
        elif kind == 0:
            g = group_of_prefill[idx]
            left[g] -= 1
            if left[g] == 0 and n >= 2:
                pending.append(dist.isend(tag((1, g, 1)), dst=dst))
        elif tok + 1 <= n - 1:
            pending.append(dist.isend(tag((1, idx, tok + 1)), dst=dst))
    for p in pending:
        p.wait()
    assert got == len(incoming), (rank, got, len(incoming))
    results[rank] = len(mine)
    dist.barrier()
    dist.destroy_process_group()


def _run(plan_json, model_json, world):
    port = _free_port()
    mgr = mp.Manager()
    res = mgr.dict()
    mp.spawn(_worker, args=(world, port, plan_json, model_json, res), nprocs=world, join=True)
    return dict(res)


def _small_plan(n=5):
    """OPT-125M-shaped 2-stage plan with eta < xi < B: several prefill
    batches and two interleaving decode groups."""
    plan = json.loads((PLANS / "opt125m_b8_1gpu.json").read_text())
    plan["workload"]["n"] = n
    plan["eta"], plan["xi"] = 2, 4
    plan["device_order"] = [0, 1]
    plan["stages"] = [{"device_index": 0, "device": "b200", "layers": [0, 5]},
                      {"device_index": 1, "device": "b200", "layers": [5, 12]}]
    o = plan["objective"]  # recompose Eq. (4) for the new (eta, xi, n)
    bc = lambda B, u: -(-(B - u) // u)
    o["total"] = (bc(8, 2) * o["t_max_pre"] + bc(8, 4) * (n - 1) * o["t_max_dec"] + o["t_pre_total"]
                  + o["t_dec_total"] + o["theta"] * o["omega_sum"])
    model = json.loads((PLANS / "opt125m_b8_1gpu.config.json").read_text())["model"]
    return json.dumps(plan), json.dumps(model)


def test_protocol_world2_interleaved_groups():
    p, m = _small_plan()
    res = _run(p, m, 2)
    assert sum(res.values()) == 2 * (4 + 2 * 4)  # each stage: 4 prefill + 2 groups x 4 tokens


@pytest.mark.parametrize("name,world", [("opt30b_b32_2gpu", 2), ("opt30b_b32_4gpu", 4),
                                        ("opt13b_b64_2gpu_weak", 2),
                                        ("opt13b_b128_4gpu_weak", 4),
                                        ("opt13b_b256_8gpu_weak", 8)])
def test_protocol_reference_plans(name, world):
    plan = (PLANS / f"{name}.json").read_text()
    model = json.dumps(json.loads((PLANS / f"{name}.config.json").read_text())["model"])
    d = json.loads(plan)
    res = _run(plan, model, world)
    B, eta, n = d["workload"]["global_bz"], d["eta"], d["workload"]["n"]
    per_stage = -(-B // eta) + -(-B // d["xi"]) * (n - 1)
    assert all(v == per_stage for v in res.values())
