mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sc_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > gpurun_out/sc_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/sc_pytest_multi.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 > gpurun_out/sc_bench_n2.json 2> gpurun_out/sc_bench_n2.err
tail -n 2 gpurun_out/sc_pytest_multi.log
