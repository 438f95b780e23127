#!/bin/bash
# round 2: N = 1 bench plain run, then its ncu launch list, then ncu --set full of the Adam kernel
# and of the rounds kernel (emulated 2x2) -- one ncu tool per call (all ncu runs count as one)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
NCU=/usr/local/cuda/bin/ncu
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_plain.json 2> gpurun_out/ncu_plain.err && \
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
python tools/ncu_adam.py > gpurun_out/ncu_adam_plain.log 2>&1 && \
$NCU --set full --clock-control none --import-source on -k regex:adam_tma -s 2 -c 1 -o gpurun_out/prof_adam_r02 \
    python tools/ncu_adam.py > gpurun_out/ncu_adam.log 2>&1
echo "adam rc=$?"
python tools/ncu_rounds.py > gpurun_out/ncu_rounds_plain.log 2>&1 && \
$NCU --set full --clock-control none --import-source on -k regex:rounds_tma -s 6 -c 2 -o gpurun_out/prof_rounds_r02 \
    python tools/ncu_rounds.py > gpurun_out/ncu_rounds.log 2>&1
echo "rounds rc=$?"
ls -la gpurun_out/*.ncu-rep
