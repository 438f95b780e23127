mkdir -p gpurun_out
for M in 1 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2954$M tools/sweep.py --model 13B --group-size $M --steps 4 --warmup 2 --grid '{"strategy":["NNN","NNI","NNG","NII","NIG","NGG","INI","ING","III","IIG","IGG","GNG","GIG","GGG"],"bucket":[536870912],"depth":[1]}' >> gpurun_out/s13_n2.jsonl 2>> gpurun_out/s13_n2.err
done
wc -l gpurun_out/s13_n2.jsonl
