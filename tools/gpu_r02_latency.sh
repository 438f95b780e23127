#!/bin/bash
# round 2: small-message all-reduce latency A/B (entry barrier, grid sizing) with the device trace
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
OUT=gpurun_out/latency_${NG}gpu.jsonl
: > $OUT
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29631 tools/coll_bench.py "$@" >> $OUT 2>> gpurun_out/latency.err; }
for EB in 1 0; do
  for CT in 0 148; do
    PARO_ENTRY_BARRIER=$EB run --sizes-mb 1,4,16,64 --topos ho,oneshot --comm-ctas $CT --iters 100 --trace --no-nccl
  done
done
run --sizes-mb 1,4,16,64,256,1024 --topos ho,oneshot --iters 20
cat $OUT
