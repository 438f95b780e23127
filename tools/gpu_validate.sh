mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r1v_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1v_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r1v_bench_n1.json 2> gpurun_out/r1v_bench_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/r1v_bench_n2.json 2> gpurun_out/r1v_bench_n2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1v_bench_ref.json 2> gpurun_out/r1v_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1v_launches_n1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r1v_ncu.log 2>&1
tail -3 gpurun_out/r1v_pytest.log
cat gpurun_out/r1v_bench_n1.json gpurun_out/r1v_bench_n2.json
