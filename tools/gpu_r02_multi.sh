#!/bin/bash
# round 2: build, selected -m gpu tests (PYTEST_K), the multi-GPU suite, bench at N = visible GPUs
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; tail -20 gpurun_out/build.log; exit 1; }
if [ -n "$PYTEST_K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -k "$PYTEST_K" > gpurun_out/pytest_k.log 2>&1; echo "pytest_k rc=$?" >> gpurun_out/pytest_k.log
  tail -8 gpurun_out/pytest_k.log
fi
if [ -z "$NO_MULTI" ]; then
  timeout 2400 python -m pytest tests/test_gpu_multi.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/pytest_multi.log 2>&1; echo "multi rc=$?" >> gpurun_out/pytest_multi.log
  tail -8 gpurun_out/pytest_multi.log
fi
if [ -z "$NO_BENCH" ]; then
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $NG ${BENCH_ARGS} > gpurun_out/bench_n$NG.json 2> gpurun_out/bench_n$NG.err; echo "bench rc=$?"
  head -c 6000 gpurun_out/bench_n$NG.json
fi
