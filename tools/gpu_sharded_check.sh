#!/bin/sh
python -m pytest tests/test_gpu_sharded.py tests/test_reference_suite_on_gpu.py -x -q 2>&1 | tail -25
python bench.py --sharded --steps 3 --warmup 1 > gpurun_out/sharded1.json 2> gpurun_out/sharded1.err; echo "sharded1 rc=$?"; tail -n 3 gpurun_out/sharded1.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --share-gpu --config c2 > gpurun_out/sharded2.json 2> gpurun_out/sharded2.err; echo "sharded2 rc=$?"; tail -n 3 gpurun_out/sharded2.err
