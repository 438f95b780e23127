#!/bin/bash
# all-reduce transport x store-path probe at large sizes (4 GPUs)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
OUT=gpurun_out/pushimpl_${NG}gpu.jsonl
: > $OUT
for tr in push pull; do for ci in tma tma_store lsu; do
echo "{\"transport\": \"$tr\", \"comm_impl\": \"$ci\"}" >> $OUT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29661 tools/coll_bench.py --sizes-mb 16,256,4096 --topos ho,flat --transport $tr --comm-impl $ci --iters 10 --no-nccl >> $OUT 2>> gpurun_out/pushimpl.err
done; done
python - <<'PY'
import json,glob
for f in glob.glob("gpurun_out/pushimpl_*gpu.jsonl"):
    for l in open(f):
        d=json.loads(l)
        if "bytes" not in d: print(d); continue
        print(d["bytes"]>>20, {k:(v["ms"],v["busbw_GBps"]) for k,v in d.items() if isinstance(v,dict)})
PY
tail -3 gpurun_out/pushimpl.err
