#!/bin/bash
# the driver's multi-GPU launch form at N=1 (torchrun, NCCL init, max-over-ranks timing)
O=gpurun_out; mkdir -p $O
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 1 --steps 5 --warmup 3 --config C1 > $O/torchrun_c1.json 2> $O/torchrun_c1.err
echo rc=$? >> $O/torchrun_c1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --impl reference --gpus 1 --steps 2 --warmup 3 --config C1 > $O/torchrun_ref_c1.json 2> $O/torchrun_ref_c1.err
echo rc=$? >> $O/torchrun_ref_c1.err
