#!/bin/bash
# torchrun path on ONE GPU (oversubscribed test mode: ranks share the device, gloo control
# collectives): strong sharding of the config's slots + IPC import of rank 0's metadata
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/multirank_strong.log 2>&1; echo "rc=$?" >> $O/multirank_strong.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --impl reference --steps 2 --warmup 3 > $O/multirank_reference.log 2>&1; echo "rc=$?" >> $O/multirank_reference.log
