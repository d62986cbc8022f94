export BT_DIST_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --steps 2 --warmup 3 --small --no-cpu > gpurun_out/dist2b.json 2> gpurun_out/dist2b.err; echo "rc=$?" >> gpurun_out/dist2b.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 2 --steps 1 --warmup 3 --no-cpu --no-extras --no-e2e > gpurun_out/dist2full.json 2> gpurun_out/dist2full.err; echo "rc=$?" >> gpurun_out/dist2full.err
