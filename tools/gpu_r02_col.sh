#!/bin/bash
# column barriers: real-rank parity (column test first, then the whole multi suite), then A/B
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "column" > gpurun_out/pytest_col.log 2>&1; rc=$?; echo "pytest_col rc=$rc head=$(cat .git_head) gpus=$NG" >> gpurun_out/pytest_col.log
tail -3 gpurun_out/pytest_col.log
[ $rc = 0 ] || { tail -60 gpurun_out/pytest_col.log; exit 1; }
OUT=gpurun_out/col_${NG}gpu.jsonl
: > $OUT
for cb in 0 1; do
echo "{\"PARO_COL_BARRIER\": $cb}" >> $OUT
PARO_COL_BARRIER=$cb timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29661 tools/coll_bench.py --sizes-mb 1,4,16,64,256,1024,4096 --topos oneshot,ho,flat --iters 20 --no-nccl >> $OUT 2>> gpurun_out/col.err
done
python - <<'PY'
import json,glob
for f in glob.glob("gpurun_out/col_*gpu.jsonl"):
    for l in open(f):
        d=json.loads(l)
        if "bytes" not in d: print(d); continue
        print(d["bytes"]>>20, {k:(v["ms"],v["busbw_GBps"]) for k,v in d.items() if isinstance(v,dict)})
PY
if [ "${FULL:-1}" = 1 ]; then
timeout 2400 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/pytest_multi.log 2>&1; echo "multi rc=$? head=$(cat .git_head) gpus=$NG" >> gpurun_out/pytest_multi.log
tail -3 gpurun_out/pytest_multi.log
fi
