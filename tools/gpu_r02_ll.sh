#!/bin/bash
# flag-in-data (LL) one-shot all-reduce: real-rank parity, then A/B vs the barrier kernel
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x -k "graph_replay or consumer or real_ranks" > gpurun_out/pytest_ll.log 2>&1; rc=$?; echo "pytest_ll rc=$rc head=$(cat .git_head) gpus=$NG" >> gpurun_out/pytest_ll.log
tail -3 gpurun_out/pytest_ll.log
[ $rc = 0 ] || { tail -80 gpurun_out/pytest_ll.log; exit 1; }
OUT=gpurun_out/ll_ab.jsonl
: > $OUT
for np in $NG 2; do
for kb in 0 4096; do
echo "{\"PARO_LL_MAX_KB\": $kb, \"ranks\": $np}" >> $OUT
PARO_LL_MAX_KB=$kb timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port 29661 tools/coll_bench.py --sizes-mb 0.25,1,2,4,16 --topos oneshot --iters 50 >> $OUT 2>> gpurun_out/ll.err
done; done
python - <<'PY'
import json
for l in open("gpurun_out/ll_ab.jsonl"):
    d=json.loads(l)
    if "bytes" not in d: print(d); continue
    print(d["bytes"]/2**20, {k:(round(v["ms"]*1000,1),v["busbw_GBps"]) for k,v in d.items() if isinstance(v,dict)})
PY
tail -3 gpurun_out/ll.err
