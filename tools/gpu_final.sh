mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fin_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/fin_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/fin_bench_n1.json 2> gpurun_out/fin_bench_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/fin_bench_n2.json 2> gpurun_out/fin_bench_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/fin_bench_n4.json 2> gpurun_out/fin_bench_n4.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 4 --impl reference --steps 3 --warmup 3 > gpurun_out/fin_bench_ref_n4.json 2> gpurun_out/fin_bench_ref_n4.err
tail -n 3 gpurun_out/fin_pytest.log; cat gpurun_out/fin_smoke.log | tail -n 2; wc -l gpurun_out/fin_bench_n*.json
