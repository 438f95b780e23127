mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fm_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fused_inter or splits_every_strategy or streamed or edge_inputs" > gpurun_out/fm_pytest_emu.log 2>&1; echo "rc=$?" >> gpurun_out/fm_pytest_emu.log
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > gpurun_out/fm_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/fm_pytest_multi.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/sweep.py --model 7B --group-size 1 --steps 6 --warmup 3 --grid '{"strategy":["NNN","NII","III"],"bucket":[536870912],"depth":[1],"fuse_allreduce":[0,1]}' > gpurun_out/fm_sweep_ab_2x1.jsonl 2> gpurun_out/fm_sweep_ab_2x1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 > gpurun_out/fm_bench_n2.json 2> gpurun_out/fm_bench_n2.err
tail -n 2 gpurun_out/fm_pytest_emu.log; tail -n 2 gpurun_out/fm_pytest_multi.log
