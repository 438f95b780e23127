#!/bin/bash
# e2e (host link) A/B of the streamed plan's bucket size, N = 1
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
OUT=gpurun_out/e2e_bucket_ab.jsonl
: > $OUT
for eb in ${EBS:-0 268435456 134217728 67108864}; do
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-bucket $eb > gpurun_out/b.json 2> gpurun_out/b.err
python - "$eb" >> $OUT <<'PY'
import json, sys
d = json.loads(open("gpurun_out/b.json").read().strip().splitlines()[-1])
e = d["e2e"]
print(json.dumps({"e2e_bucket_arg": int(sys.argv[1]), "bucket_elems": e.get("bucket_elems"), "ms_params_back": round(e["ms_per_step"], 2),
                  "pcie_GBps": round(e["pcie_GBps_per_gpu"], 1), "ms_stats_only": round(e["stats_only"]["ms_per_step"], 2), "step_ms": round(d["ms_per_step"], 3)}))
PY
done
cat $OUT
