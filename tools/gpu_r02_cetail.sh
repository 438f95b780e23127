#!/bin/bash
# copy-engine tails (copy_engine = 3): real-rank parity + graph replay, then the all-reduce sweep
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x -k "ce_tails or graph_replay" > gpurun_out/pytest_cetail.log 2>&1; echo "pytest rc=$? head=$(cat .git_head) gpus=$NG" >> gpurun_out/pytest_cetail.log
tail -3 gpurun_out/pytest_cetail.log
OUT=gpurun_out/cetail_${NG}gpu.jsonl
: > $OUT
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29661 tools/coll_bench.py --sizes-mb ${SIZES:-16,64,256,1024,4096} --topos ho,ho+ce,oneshot,oneshot+ce,flat+ce --iters 10 >> $OUT 2>> gpurun_out/cetail.err
python - <<'PY'
import json,glob
for f in glob.glob("gpurun_out/cetail_*gpu.jsonl"):
    for l in open(f):
        d=json.loads(l)
        print(d["bytes"]>>20, {k:(v["ms"],v["busbw_GBps"]) for k,v in d.items() if isinstance(v,dict)})
PY
tail -5 gpurun_out/cetail.err
