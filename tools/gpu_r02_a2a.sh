#!/bin/bash
# round 2: why one-shot (all-to-all) pulls are slower than rings at medium/large sizes (4 GPUs)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_n1_c.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_n1_c.json')); print(d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel'], d['clocks'])"
OUT=gpurun_out/a2a_${NG}gpu.jsonl
: > $OUT
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29651 tools/coll_bench.py "$@" >> $OUT 2>> gpurun_out/a2a.err; }
for ST in 0 8; do
  for OP in ar ag; do
    PARO_RT_STAGES=$ST PARO_ONESHOT_MAX_MB=8192 run --op $OP --sizes-mb 16,64,256 --topos ho,oneshot,direct --iters 20 --trace --no-nccl
  done
done
cat $OUT | cut -c1-400
