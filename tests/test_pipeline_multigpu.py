"""Multi-GPU pipeline parity (needs >= 2 / 4 GPUs; run with `gpurun --gpus N`):
a plan executed over N processes / N B200s with NCCL P2P (hidden states
forward, next-token ids fed back from the last stage to stage 0) must
produce generated tokens and final hidden states bit-identical to the same
plan run as ONE stage on one GPU (same kernels, same grids, same order per
layer). Plans: an OPT-125M-shaped plan cut into 2 / 4 stages with two
interleaving decode groups, and the reference planner's OPT-30B 2- and
4-stage partitions (tests/golden/plans/opt30b_b32_{2,4}gpu.json,
optimizer_planner.cpp:79-170, BASELINE configs[2])."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
PLANS = ROOT / "tests" / "golden" / "plans"

WORKER = r'''
import json, os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.environ["HP_ROOT"])
from paper_2403_01136_b200.pipeline import Pipeline, nccl_ids
from tests.test_pipeline_multigpu import _plan
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
plan, model = _plan(os.environ["HP_PLAN"], world)
B, n, h1 = plan["workload"]["global_bz"], plan["workload"]["n"], int(os.environ["HP_H1"])
obj = [nccl_ids(world) if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
p = Pipeline(json.dumps(plan), model, rank, world, obj[0], sm_budget=140, timeout_s=120)
out = torch.empty(B * n, dtype=torch.int32).pin_memory()
for _ in range(2):
    p.run(None, out.data_ptr() if rank == world - 1 else None)
if rank == world - 1:
    hid = torch.empty(B * h1, dtype=torch.bfloat16)
    p.final_hidden(hid.data_ptr())
    torch.save((out.clone(), hid), os.environ["HP_OUT"])
p.close()
dist.barrier()
'''


def _plan(name, world):
    """(plan dict with `world` stages, model JSON) for a case name."""
    if name == "small":
        from tests.test_pipeline_protocol import _small_plan
        plan, model = _small_plan(n=6)
        plan = json.loads(plan)
        cut = [round(12 * j / world) for j in range(world + 1)]
        plan["device_order"] = list(range(world))
        plan["stages"] = [{"device_index": j, "device": "b200", "layers": [cut[j], cut[j + 1]]}
                          for j in range(world)]
        return plan, model
    plan = json.loads((PLANS / f"{name}.json").read_text())
    model = json.dumps(json.loads((PLANS / f"{name}.config.json").read_text())["model"])
    plan["workload"]["n"] = 3  # xi == B: the objective does not depend on n
    if world == 1:
        L = plan["num_layers"]
        plan["device_order"], plan["devices"] = [0], plan["devices"][:1]
        plan["stages"] = [{"device_index": 0, "device": "b200", "layers": [0, L]}]
    else:
        assert len(plan["stages"]) == world
    return plan, model


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,world,h1", [("small", 2, 768), ("small", 4, 768),
                                           ("opt30b_b32_2gpu", 2, 7168),
                                           ("opt30b_b32_4gpu", 4, 7168)])
def test_multistage_pipeline_bit_identical_to_single_gpu(cuda, tmp_path, name, world, h1):
    import torch
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2403_01136_b200.pipeline import Pipeline
    one, model = _plan(name, 1)
    B, n = one["workload"]["global_bz"], one["workload"]["n"]
    p = Pipeline(json.dumps(one), model, sm_budget=140, timeout_s=120)
    ref = torch.empty(B * n, dtype=torch.int32).pin_memory()
    for _ in range(2):
        p.run(None, ref.data_ptr())
    ref_hid = torch.empty(B * h1, dtype=torch.bfloat16)
    p.final_hidden(ref_hid.data_ptr())
    p.close()
    torch.cuda.empty_cache()
    w = tmp_path / "w.py"
    w.write_text(WORKER)
    outp = tmp_path / "out.pt"
    env = dict(os.environ, HP_ROOT=str(ROOT), HP_OUT=str(outp), HP_PLAN=name, HP_H1=str(h1))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
                        f"--master-port={_port()}", str(w)], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    got, hid = torch.load(outp)
    assert torch.isfinite(hid.float()).all()
    assert torch.equal(got, ref)
    assert torch.equal(hid, ref_hid)
