# round-2 session l: bench.py under torchrun with 2 ranks sharing the one GPU (gloo collectives; the ranks'
# kernels never wait on each other): the normal path, then the sub-record watchdog forced to fire
set -x
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
HSGN_BENCH_BACKEND=gloo timeout 600 $TR --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu --members 1024 > gpurun_out/r02l_bench2.json 2> gpurun_out/r02l_bench2.err; echo "bench2 rc $?"
HSGN_BENCH_SUB_TIMEOUT=0.01 HSGN_BENCH_BACKEND=gloo timeout 600 $TR --master-port 29512 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu --members 1024 > gpurun_out/r02l_bench2_wd.json 2> gpurun_out/r02l_bench2_wd.err; echo "bench2 watchdog rc $?"
wc -l gpurun_out/r02l_bench2.json gpurun_out/r02l_bench2_wd.json
tail -c 300 gpurun_out/r02l_bench2.json; echo; tail -c 300 gpurun_out/r02l_bench2_wd.json; echo
tail -3 gpurun_out/r02l_bench2.err gpurun_out/r02l_bench2_wd.err
