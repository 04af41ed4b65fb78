set -x
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for c in C3 C6; do timeout 600 python bench.py --config $c > gpurun_out/b_${c}_g1.json 2> gpurun_out/b_${c}_g1.err; done
for n in 2 4; do for c in C4 C3 C6; do timeout 600 $R --nproc-per-node $n --master-port 2950$n bench.py --gpus $n --config $c > gpurun_out/b_${c}_g$n.json 2> gpurun_out/b_${c}_g$n.err; done; done
timeout 600 python bench.py --config C5 > gpurun_out/b_C5_g1.json 2> gpurun_out/b_C5_g1.err
echo done
