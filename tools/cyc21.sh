BENCH_BACKEND=gloo timeout -k 5 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/b2.log 2>&1; echo rc $?; tail -c 1500 gpurun_out/b2.log
timeout -k 5 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
