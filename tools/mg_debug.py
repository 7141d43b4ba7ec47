"""2-rank pipeline smoke with progress logging (debug the NCCL path).
  torchrun --nproc-per-node 2 tools/mg_debug.py <pdl 0/1> <graphs 0/1>"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def log(*a):
    print(f"[rank {os.environ.get('RANK')}] {time.strftime('%X')}", *a, file=sys.stderr, flush=True)


def main():
    import torch
    import torch.distributed as dist
    from paper_2403_01136_b200 import capi
    from paper_2403_01136_b200.pipeline import Pipeline, nccl_ids
    from tests.test_pipeline_protocol import _small_plan
    pdl, graphs = int(sys.argv[1]), int(sys.argv[2])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    capi.lib.hp_set_pdl(pdl)
    dist.init_process_group("gloo")
    plan, model = _small_plan(n=3)
    obj = [nccl_ids(world) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    log("creating pipeline")
    p = Pipeline(plan, model, rank, world, obj[0], sm_budget=140, use_graphs=bool(graphs),
                 timeout_s=float(os.environ.get('HP_TIMEOUT', '40')))
    log("created; info", p.info())
    for i in range(2):
        try:
            t = p.run()
        except Exception as e:  # noqa: BLE001
            log("run", i, "FAILED", repr(e))
            os._exit(3)
        log("run", i, "done", t)
    p.close()
    dist.barrier()
    log("ok")


if __name__ == "__main__":
    main()
