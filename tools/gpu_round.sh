# full GPU check: tests, smoke, bench (N=1), functional N=2 bench over gloo on one GPU
python -m pytest tests -m gpu -q -x --tb=short > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; tail -c 400 gpurun_out/bench.log
BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2.log 2>&1; tail -c 600 gpurun_out/bench_n2.log
