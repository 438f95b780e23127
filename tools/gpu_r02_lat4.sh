#!/bin/bash
# round 2: multi-GPU suite, latency sweep (entry barrier on, auto grid) and bench at N = visible GPUs
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
if [ -z "$NO_MULTI" ]; then
  timeout 2400 python -m pytest tests/test_gpu_multi.py -m gpu -q -rs > gpurun_out/pytest_multi_${NG}gpu.log 2>&1; echo "multi rc=$? head=$(cat .git_head)" >> gpurun_out/pytest_multi_${NG}gpu.log
  tail -4 gpurun_out/pytest_multi_${NG}gpu.log
fi
OUT=gpurun_out/latency_${NG}gpu.jsonl
: > $OUT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29631 tools/coll_bench.py --sizes-mb 1,4,16,64 --topos ho,oneshot --iters 100 --trace --no-nccl >> $OUT 2>> gpurun_out/latency.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29632 tools/coll_bench.py --sizes-mb 1,4,16,64,256,1024,4096 --topos ho,oneshot --iters 20 >> $OUT 2>> gpurun_out/latency.err
cat $OUT | cut -c1-400
if [ -z "$NO_BENCH" ]; then
  timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $NG ${BENCH_ARGS} > gpurun_out/bench_n$NG.json 2> gpurun_out/bench_n$NG.err; echo "bench rc=$?"
  head -c 600 gpurun_out/bench_n$NG.json
fi
