export PFB_BENCH_BACKEND=gloo
for c in cfg4 cfg5; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus 2 --steps 3 --warmup 3 --config $c --no-cpu-baseline 2>&1 | grep -E '^\{|Error|error' | cut -c1-300
done
