#!/bin/bash
# BASELINE config 4 (LLaMA-30B list, OS = G strategies) at 2x2 with streamed gradients (grad_slots = 4,
# a copy producer inside the timed step), round-2 kernels
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
OUT=gpurun_out/sweep30b_2x2_r02.jsonl
: > $OUT
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 tools/sweep.py --model 30B --group-size 2 --steps 3 --warmup 2 --mem-cap-gb 175 --grid '{"strategy":["NNG","NIG","NGG","ING","IIG","IGG","GNG","GIG","GGG"],"bucket":[268435456],"depth":[2],"comm_ctas":[0],"comm_impl":["tma"],"grad_slots":[4],"producer":["copy"]}' >> $OUT 2>> gpurun_out/s30.err
python - <<'PY'
import json
for l in open("gpurun_out/sweep30b_2x2_r02.jsonl"):
    d = json.loads(l)
    print(d.get("groups"), d["cfg"]["strategy"], d.get("ms"), d.get("Gparam_s"), d.get("footprint_gb"), d.get("skipped", ""))
PY
tail -3 gpurun_out/s30.err
