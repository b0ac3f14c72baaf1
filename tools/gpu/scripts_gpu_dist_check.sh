#!/bin/bash
# functional check of the multi-GPU bench path on ONE GPU: 2 ranks on cuda:0 over gloo
mkdir -p gpurun_out
python -c "from paper_2504_08009_b200 import build; build.build()" > gpurun_out/build.log 2>&1
for extra in "--chunks 1" "--chunks 3" "--chunks 2 --mode accu"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 2 --warmup 3 --size 2048 --dist-backend gloo --no-e2e --no-context --no-cpu-baseline $extra \
    > gpurun_out/dist_check.json 2> gpurun_out/dist_check.err; echo "dist check [$extra] rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/dist_check.json')); print(d['value'], d['compwise_err'], d['max_rel_err'], d['config']['workload'])"; grep -i error gpurun_out/dist_check.err | tail -3
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --steps 2 --warmup 3 --size 2048 --k 4096 --dist-backend gloo --parallel ksplit --no-e2e --no-context --no-cpu-baseline \
  > gpurun_out/dist_check.json 2> gpurun_out/dist_check.err; echo "dist check [ksplit] rc=$?"
python -c "import json; d=json.load(open('gpurun_out/dist_check.json')); print(d['value'], d['compwise_err'], d['max_rel_err'], d['config']['workload'], d['config']['parallelism'], d['scaling'])"; grep -i error gpurun_out/dist_check.err | tail -3
