# bench.py N=2 through torchrun on one B200 with SW_BENCH_BACKEND=gloo (both ranks share the GPU): a functional
# check of the request-sharded line (per-GPU arrival rate kept, gather/fold), not a scaling number
mkdir -p gpurun_out
for wl in tiny 8b-poisson; do
  SW_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 2 --steps 1 --warmup 3 --workload $wl > gpurun_out/multirank_$wl.log 2>&1
  echo "$wl rc=$?"
  grep '^{' gpurun_out/multirank_$wl.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['value'], d['config']['arrival'], d['config']['arrival_global'], d['split']['requests'], d['split_over_best_serial'])"
done
