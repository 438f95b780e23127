#!/bin/bash
# round 2: warp-specialized Adam A/B at N = 1 (alternating), parity subset with it on
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
PARO_ADAM_WS=1 timeout 1200 python -m pytest tests -m gpu -q -k "n1_ten or 4m_2x4_ten or variant_selection or fp32 or oneshot or consumer or streamed_step_every" > gpurun_out/pytest_ws.log 2>&1; echo "pytest_ws rc=$?" >> gpurun_out/pytest_ws.log
tail -3 gpurun_out/pytest_ws.log
: > gpurun_out/ws_ab.jsonl
for i in 1 2 3; do
  for W in 0 1; do
    PARO_ADAM_WS=$W timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print(json.dumps({'ws': $W, 'ms': d['ms_per_step'], 'frac': d['roofline']['frac'], 'kernel': d['roofline']['kernel'], 'clk': d['clocks']}))" >> gpurun_out/ws_ab.jsonl
  done
done
cat gpurun_out/ws_ab.jsonl
