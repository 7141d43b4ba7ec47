"""Multi-GPU pipeline parity (needs >= 2 GPUs; run with `gpurun --gpus 2`):
a 2- (4-) stage OPT-125M-shaped plan executed over 2 processes / 2 B200s with
NCCL P2P (hidden states forward, next-token ids fed back from the last
stage to stage 0) must produce generated tokens and final hidden states
bit-identical to the same plan run as one stage on one GPU (same kernels,
same order per layer)."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

WORKER = r'''
import json, os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.environ["HP_ROOT"])
from paper_2403_01136_b200.pipeline import Pipeline, nccl_ids
from tests.test_pipeline_protocol import _small_plan
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
plan, model = _small_plan(n=6)
plan = json.loads(plan)
cut = [round(12 * j / world) for j in range(world + 1)]
plan["device_order"] = list(range(world))
plan["stages"] = [{"device_index": j, "device": "b200", "layers": [cut[j], cut[j + 1]]}
                  for j in range(world)]
obj = [nccl_ids(world) if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
p = Pipeline(json.dumps(plan), model, rank, world, obj[0], sm_budget=140, timeout_s=60)
out = torch.empty(8 * 6, dtype=torch.int32).pin_memory()
for _ in range(2):
    p.run(None, out.data_ptr() if rank == world - 1 else None)
if rank == world - 1:
    hid = torch.empty(8 * 768, dtype=torch.bfloat16)
    p.final_hidden(hid.data_ptr())
    torch.save((out.clone(), hid), os.environ["HP_OUT"])
p.close()
dist.barrier()
'''


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
def test_multistage_pipeline_bit_identical_to_single_gpu(cuda, tmp_path, world):
    import torch
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2403_01136_b200.pipeline import Pipeline
    from tests.test_pipeline_protocol import _small_plan
    plan, model = _small_plan(n=6)
    one = json.loads(plan)
    one["device_order"] = [0]
    one["stages"] = [{"device_index": 0, "device": "b200", "layers": [0, 12]}]
    p = Pipeline(json.dumps(one), model, sm_budget=140, timeout_s=60)
    ref = torch.empty(8 * 6, dtype=torch.int32).pin_memory()
    for _ in range(2):
        p.run(None, ref.data_ptr())
    ref_hid = torch.empty(8 * 768, dtype=torch.bfloat16)
    p.final_hidden(ref_hid.data_ptr())
    p.close()
    w = tmp_path / "w.py"
    w.write_text(WORKER)
    outp = tmp_path / "out.pt"
    env = dict(os.environ, HP_ROOT=str(ROOT), HP_OUT=str(outp))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
                        f"--master-port={_port()}", str(w)], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-4000:]
    got, hid = torch.load(outp)
    assert torch.isfinite(hid.float()).all()
    assert torch.equal(got, ref)
    assert torch.equal(hid, ref_hid)
