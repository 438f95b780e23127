#!/bin/bash
# round 2 final (4 GPUs): fp32-wire accumulation parity, push-transport all-reduce probe, bench N = 4
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -k "fp32_wire_accumulation or oneshot or consumer" > gpurun_out/pytest_k.log 2>&1; echo "pytest_k rc=$? head=$(cat .git_head)" >> gpurun_out/pytest_k.log
tail -3 gpurun_out/pytest_k.log
OUT=gpurun_out/push_${NG}gpu.jsonl
: > $OUT
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29661 tools/coll_bench.py --sizes-mb 64,256,1024,4096 --topos ho,flat --transport push --iters 10 >> $OUT 2>> gpurun_out/push.err
cat $OUT | cut -c1-300
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $NG > gpurun_out/bench_n$NG.json 2> gpurun_out/bench_n$NG.err; echo "bench rc=$?"
head -c 400 gpurun_out/bench_n$NG.json
