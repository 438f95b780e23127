#!/bin/bash
# collective-only launches with 200 KB TMA stages (16 KB slots): parity, then A/B vs the 96 KB co-run stages
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "collective" > gpurun_out/pytest_solo.log 2>&1; echo "pytest rc=$? head=$(cat .git_head)" >> gpurun_out/pytest_solo.log
tail -3 gpurun_out/pytest_solo.log
OUT=gpurun_out/solo_${NG}gpu.jsonl
: > $OUT
for solo in 0 1 default; do
echo "{\"PARO_RT_SOLO\": \"$solo\"}" >> $OUT
if [ $solo = default ]; then unset PARO_RT_SOLO; else export PARO_RT_SOLO=$solo; fi
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29661 tools/coll_bench.py --sizes-mb ${SIZES:-1,4,16,64,256,1024,4096} --topos oneshot,ho,flat --iters 20 --no-nccl >> $OUT 2>> gpurun_out/solo.err
done
unset PARO_RT_SOLO
python - <<'PY'
import json,glob
for f in glob.glob("gpurun_out/solo_*gpu.jsonl"):
    for l in open(f):
        d=json.loads(l)
        if "bytes" not in d: print(d); continue
        print(d["bytes"]>>20, {k:(v["ms"],v["busbw_GBps"]) for k,v in d.items() if isinstance(v,dict)})
PY
tail -3 gpurun_out/solo.err
