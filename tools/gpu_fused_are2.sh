mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fb_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fused_inter or accumulation or splits_every_strategy or streamed or clipping or edge_inputs or ten_steps" > gpurun_out/fb_pytest_emu.log 2>&1; echo "rc=$?" >> gpurun_out/fb_pytest_emu.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider > gpurun_out/fb_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/fb_pytest_multi.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 tools/sweep.py --model 7B --group-size 2 --steps 6 --warmup 3 --grid '{"strategy":["INI","NNI"],"bucket":[536870912],"depth":[1],"fuse_allreduce":[0,1]}' > gpurun_out/fb_sweep_ab_2x2.jsonl 2> gpurun_out/fb_sweep_ab_2x2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 4 > gpurun_out/fb_bench_n4.json 2> gpurun_out/fb_bench_n4.err
tail -n 2 gpurun_out/fb_pytest_emu.log; tail -n 2 gpurun_out/fb_pytest_multi.log; tail -c 600 gpurun_out/fb_bench_n4.err
