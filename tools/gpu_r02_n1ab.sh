#!/bin/bash
# round 2: N = 1 A/B of Adam L2 eviction hints (alternating runs), then the ncu job
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/n1_ab.jsonl
for i in 1 2; do
  for H in 0 1; do
    PARO_L2_HINT=$H timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/ab.json')); print(json.dumps({'l2_hint': $H, 'ms': d['ms_per_step'], 'frac': d['roofline']['frac'], 'kernel': d['roofline']['kernel'], 'clk': d['clocks']}))" >> gpurun_out/n1_ab.jsonl
  done
done
cat gpurun_out/n1_ab.jsonl
if [ -z "$NO_NCU" ]; then bash tools/gpu_r02_ncu.sh; fi
