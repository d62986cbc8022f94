# N > 1 bench path on one GPU: ranks stacked on GPU 0 with the gloo test hook
export BT_DIST_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --small --no-cpu > gpurun_out/dist2.json 2> gpurun_out/dist2.err; echo "rc=$?" >> gpurun_out/dist2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 3 --steps 2 --warmup 3 --small --no-cpu --no-extras > gpurun_out/dist3.json 2> gpurun_out/dist3.err; echo "rc=$?" >> gpurun_out/dist3.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/ref2.json 2> gpurun_out/ref2.err; echo "rc=$?" >> gpurun_out/ref2.err
