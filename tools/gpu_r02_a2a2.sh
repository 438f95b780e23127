#!/bin/bash
# round 2: one-shot after the rotated peer order; slot size A/B for nested folds (4 GPUs)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
OUT=gpurun_out/a2a2_${NG}gpu.jsonl
: > $OUT
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29651 tools/coll_bench.py "$@" >> $OUT 2>> gpurun_out/a2a.err; }
for LG in 0 12; do
  PARO_RT_SLOT_LG=$LG PARO_ONESHOT_MAX_MB=8192 run --op ar --sizes-mb 4,16,64,256,1024 --topos ho,oneshot --iters 20 --trace
done
PARO_ONESHOT_MAX_MB=8192 run --op ag --sizes-mb 16,64,256 --topos ho,oneshot --iters 20 --trace --no-nccl
cat $OUT | cut -c1-300
