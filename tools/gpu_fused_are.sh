mkdir -p gpurun_out
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fa_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fused_inter or splits_every_strategy or ten_steps or edge_inputs" > gpurun_out/fa_pytest_emu.log 2>&1; echo "rc=$?" >> gpurun_out/fa_pytest_emu.log
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > gpurun_out/fa_pytest_multi.log 2>&1; echo "rc=$?" >> gpurun_out/fa_pytest_multi.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tools/sweep.py --model 7B --group-size 2 --steps 6 --warmup 3 --grid '{"strategy":["NNN","NNI","NNG","NII","NIG","NGG","INI","ING","III","IIG","IGG","GNG","GIG","GGG"],"bucket":[536870912],"depth":[1]}' > gpurun_out/fa_sweep_all_2x2.jsonl 2> gpurun_out/fa_sweep_all_2x2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 tools/sweep.py --model 7B --group-size 2 --steps 6 --warmup 3 --grid '{"strategy":["III","NII"],"bucket":[536870912],"depth":[1],"fuse_allreduce":[0,1]}' > gpurun_out/fa_sweep_ab_2x2.jsonl 2> gpurun_out/fa_sweep_ab_2x2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 4 > gpurun_out/fa_bench_n4.json 2> gpurun_out/fa_bench_n4.err
tail -2 gpurun_out/fa_pytest_emu.log gpurun_out/fa_pytest_multi.log
