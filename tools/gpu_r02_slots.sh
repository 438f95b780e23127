#!/bin/bash
# one-shot all-reduce: nested-fold slot size A/B (PARO_RT_SLOT_LG), medium sizes
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
OUT=gpurun_out/slots_${NG}gpu.jsonl
: > $OUT
for lg in 13 12 11; do
echo "{\"PARO_RT_SLOT_LG\": $lg}" >> $OUT
PARO_RT_SLOT_LG=$lg timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29661 tools/coll_bench.py --sizes-mb 4,16,64,256 --topos oneshot,ho --iters 20 --no-nccl >> $OUT 2>> gpurun_out/slots.err
done
python - <<'PY'
import json,glob
for f in glob.glob("gpurun_out/slots_*gpu.jsonl"):
    for l in open(f):
        d=json.loads(l)
        if "bytes" not in d: print(d); continue
        print(d["bytes"]>>20, {k:(v["ms"],v["busbw_GBps"]) for k,v in d.items() if isinstance(v,dict)})
PY
