# N>1: persistent-grid SM budget next to NCCL's P2P kernels (2 channels per link)
N=$(nvidia-smi -L | wc -l)
for b in 140 144 146 148; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --steps 3 --warmup 3 --sm-budget $b > gpurun_out/r2_smb_$b.log 2>&1
  echo "budget $b rc=$? $(grep '^{' gpurun_out/r2_smb_$b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],1))')"
done
