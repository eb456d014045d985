# the bench's non-default workloads at HEAD: configs[1] (1b) and configs[4] (8b-long)
mkdir -p gpurun_out
timeout 600 python bench.py --workload 1b --steps 3 --warmup 3 > gpurun_out/bench_1b.log 2>&1; echo "1b rc=$?"
timeout 1500 python bench.py --workload 8b-long --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_8b_long.log 2>&1; echo "8b-long rc=$?"
for f in gpurun_out/bench_1b.log gpurun_out/bench_8b_long.log; do
grep '^{' $f | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['config']['workload'], d['value'], d['split_over_best_serial'], d.get('chunked') and d['chunked']['tokens_per_s'], d['roofline']['frac'], d['roofline'].get('after_prefill',{}).get('frac'), d.get('roofline_decode_step') and d['roofline_decode_step']['frac'], d['reference_simulator'] and d['reference_simulator'].get('simulated_split_over_serial'))"
done
