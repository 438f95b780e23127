#!/bin/bash
# BASELINE config 3 (LLaMA-13B list) at 2 GPUs, every split and every strategy that fits, round-2 defaults
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
OUT=gpurun_out/sweep13b_n2_r02.jsonl
: > $OUT
for M in 1 2; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2955$M tools/sweep.py --model 13B --group-size $M --steps 4 --warmup 2 --mem-cap-gb 170 --grid '{"strategy":["NNN","NNI","NNG","NII","NIG","NGG","INI","ING","III","IIG","IGG","GNG","GIG","GGG"],"bucket":[536870912],"depth":[1],"comm_ctas":[0],"copy_engine":[1]}' >> $OUT 2>> gpurun_out/s13.err
done
python - <<'PY'
import json
for l in open("gpurun_out/sweep13b_n2_r02.jsonl"):
    d = json.loads(l)
    print(d.get("groups"), d["cfg"]["strategy"], d.get("ms"), d.get("Gparam_s"), d.get("footprint_gb"), d.get("skipped", ""))
PY
tail -3 gpurun_out/s13.err
