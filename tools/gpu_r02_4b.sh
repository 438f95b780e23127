#!/bin/bash
# round 2 (4 GPUs): multi-GPU suite, small-message micro-sweep with traces, IIG copy-engine sweep, bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 2400 python -m pytest tests/test_gpu_multi.py -m gpu -q -rs -x > gpurun_out/pytest_multi_${NG}gpu.log 2>&1; echo "multi rc=$? head=$(cat .git_head)" >> gpurun_out/pytest_multi_${NG}gpu.log
tail -4 gpurun_out/pytest_multi_${NG}gpu.log
OUT=gpurun_out/latency_${NG}gpu_b.jsonl
: > $OUT
for CT in 0 64 148; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29631 tools/coll_bench.py --sizes-mb 1,4,16 --topos ho,oneshot,direct --comm-ctas $CT --iters 100 --trace --no-nccl >> $OUT 2>> gpurun_out/latency.err
done
cat $OUT | cut -c1-300
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29641 tools/sweep.py --grid '{"strategy":["IIG"],"copy_engine":[0,1,2],"bucket":[536870912],"depth":[1]}' > gpurun_out/sweep_ce_${NG}gpu.jsonl 2> gpurun_out/sweep.err
cat gpurun_out/sweep_ce_${NG}gpu.jsonl | cut -c1-300
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $NG ${BENCH_ARGS} > gpurun_out/bench_n$NG.json 2> gpurun_out/bench_n$NG.err; echo "bench rc=$?"
head -c 600 gpurun_out/bench_n$NG.json
