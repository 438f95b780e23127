#!/bin/bash
# round 2: build, selected -m gpu tests (PYTEST_K), then ONE compute-sanitizer tool (TOOL) on smoke()
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo build failed; tail -20 gpurun_out/build.log; exit 1; }
if [ -n "$PYTEST_K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -k "$PYTEST_K" > gpurun_out/pytest_k.log 2>&1; echo "pytest_k rc=$?" >> gpurun_out/pytest_k.log
  tail -8 gpurun_out/pytest_k.log
fi
if [ -n "$TOOL" ]; then
  timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_plain.log 2>&1 && \
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $TOOL --target-processes all ${SAN_ARGS} \
     python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/sanitizer_$TOOL.log 2>&1
  echo "sanitizer $TOOL rc=$?"
  tail -15 gpurun_out/sanitizer_$TOOL.log
fi
