# every workload's bench line at HEAD (1 x B200)
mkdir -p gpurun_out/allcfg
for W in tiny 1b 8b-poisson; do timeout 900 python bench.py --workload $W --no-cpu-baseline > gpurun_out/allcfg/$W.jsonl 2> gpurun_out/allcfg/$W.err; echo "$W rc=$?"; done
timeout 1500 python bench.py --workload 8b-long --steps 1 --no-cpu-baseline > gpurun_out/allcfg/8b-long.jsonl 2> gpurun_out/allcfg/8b-long.err; echo "8b-long rc=$?"
for W in tiny 1b 8b-poisson 8b-long; do python -c "
import json;d=json.loads(open('gpurun_out/allcfg/$W.jsonl').read().strip().splitlines()[-1])
print('$W', d['value'], d['split_over_best_serial'], d['split']['p50_ttft_s'], d['split']['p50_tbt_s'], d['roofline']['kernel'][:40], d['roofline']['frac'], (d.get('chunked') or {}).get('tokens_per_s'))"; done
