# the N > 1 sharded bench path on the single-GPU box: a 1-rank NCCL group (C4, C5)
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --mode sharded --config C4 --steps 5 --warmup 3 > gpurun_out/sh_c4_n1.log 2>&1
