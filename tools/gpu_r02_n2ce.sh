#!/bin/bash
# N = 2 (2x1) IIG: parameter gathers fused into Adam (SM pushes) vs on the copy engines
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
OUT=gpurun_out/n2_ce_ab.jsonl
: > $OUT
for cfg in "auto gathers" "never gathers" "never off" "auto gathers"; do
set -- $cfg
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 10 --fuse-gather $1 --copy-engine $2 --no-e2e --no-cpu-baseline --no-ho-ring --strategy-steps 0 > gpurun_out/b2.json 2> gpurun_out/b2.err
python - "$1" "$2" >> $OUT <<'PY'
import json, sys
d = json.loads(open("gpurun_out/b2.json").read().strip().splitlines()[-1])
print(json.dumps({"fuse_gather": sys.argv[1], "copy_engine": sys.argv[2], "ms": round(d["ms_per_step"], 3),
                  "Gparam_s": round(d["value"] / 1e9, 1), "step_frac": round(d["step_roofline"]["frac"], 3)}))
PY
done
cat $OUT
