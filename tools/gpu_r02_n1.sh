#!/bin/bash
# round 2: Adam-path parity subset + smoke + N = 1 bench (x2) + the ncu job
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -k "${PYTEST_K:-n1_ten or 4m_2x4_ten or variant_selection or fp32 or fused_inter or consumer}" > gpurun_out/pytest_k.log 2>&1; echo "pytest_k rc=$?" >> gpurun_out/pytest_k.log
tail -4 gpurun_out/pytest_k.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -6 gpurun_out/smoke.log
for i in 1 2; do
  timeout 900 python bench.py > gpurun_out/bench_n1_$i.json 2> gpurun_out/bench_n1_$i.err; echo "bench rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/bench_n1_$i.json')); print(d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel'], d['clocks'], d['e2e']['ms_per_step'])"
done
if [ -z "$NO_NCU" ]; then bash tools/gpu_r02_ncu.sh; fi
