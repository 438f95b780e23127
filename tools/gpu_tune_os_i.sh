mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 tools/sweep.py --model 7B --group-size 2 --steps 6 --warmup 3 --grid '{"strategy":["III","INI","IIG"],"bucket":[268435456,536870912],"depth":[1],"comm_ctas":[74,148]}' > gpurun_out/tu_7b_2x2.jsonl 2> gpurun_out/tu_7b_2x2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29552 tools/sweep.py --model 13B --group-size 2 --steps 4 --warmup 2 --grid '{"strategy":["NNI","NII","INI","III","IIG","GGG"],"bucket":[536870912],"depth":[1]}' > gpurun_out/tu_13b_2x2.jsonl 2> gpurun_out/tu_13b_2x2.err
wc -l gpurun_out/tu_*.jsonl
