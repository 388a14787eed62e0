
VF_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --side 256 --steps 2 --warmup 1 > gpurun_out/sharded2.json 2> gpurun_out/sharded2.err
VF_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --side 256 --steps 2 --warmup 1 > gpurun_out/sharded4.json 2> gpurun_out/sharded4.err
