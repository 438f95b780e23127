mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 tools/sweep.py --model 7B --group-size 2 --steps 6 --warmup 3 --grid '{"strategy":["III","INI","IIG"],"bucket":[536870912],"depth":[1],"adam_impl":["auto","tma_store"]}' > gpurun_out/as_2x2.jsonl 2> gpurun_out/as_2x2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 tools/sweep.py --model 7B --group-size 1 --steps 6 --warmup 3 --grid '{"strategy":["NNN","III","IIG","GGG"],"bucket":[536870912],"depth":[1],"adam_impl":["auto","tma_store"]}' > gpurun_out/as_2x1.jsonl 2> gpurun_out/as_2x1.err
wc -l gpurun_out/as_*.jsonl
