#!/bin/bash
# round 2: build, the COMPLETE -m gpu suite on every visible GPU, smoke, bench at N = visible GPUs
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
git_head=$(cat .git_head 2>/dev/null)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; tail -20 gpurun_out/build.log; exit 1; }
timeout 3000 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_full_${NG}gpu.log 2>&1; echo "pytest rc=$? head=$git_head gpus=$NG" >> gpurun_out/pytest_full_${NG}gpu.log
tail -12 gpurun_out/pytest_full_${NG}gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ -z "$NO_BENCH" ]; then
  if [ "$NG" = "1" ]; then
    timeout 1200 python bench.py ${BENCH_ARGS} > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench rc=$?"
  else
    timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $NG ${BENCH_ARGS} > gpurun_out/bench_n$NG.json 2> gpurun_out/bench_n$NG.err; echo "bench rc=$?"
  fi
  head -c 1500 gpurun_out/bench_n$NG.json
fi
if [ -n "$ALSO_N2" ] && [ "$NG" -ge 2 ]; then
  CUDA_VISIBLE_DEVICES=0,1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 ${BENCH_ARGS} > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench n2 rc=$?"
  head -c 600 gpurun_out/bench_n2.json
fi
