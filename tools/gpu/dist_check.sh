#!/bin/bash
# Functional check of the multi-GPU bench path on a 1-GPU box: 2 ranks on cuda:0
# over gloo (NCCL refuses two ranks on one device), row-block strong scaling with
# the column-panel broadcast and per-panel gather.  Numbers are NOT bench values.
mkdir -p gpurun_out
N=${N:-4096}
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
   --master-port 29511 bench.py --gpus 2 --steps 1 --warmup 3 --dist-backend gloo --size $N --acc-samples 64 \
   > gpurun_out/dist_check_$N.json 2> gpurun_out/dist_check_$N.err
echo "dist check n=$N rc=$?"; tail -c 1500 gpurun_out/dist_check_$N.json; tail -5 gpurun_out/dist_check_$N.err
