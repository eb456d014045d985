# bench A/B of an env toggle on one box: bash tools/gpu/bench_ab.sh VAR v1 v2
mkdir -p gpurun_out
for V in $2 $3 $2 $3; do
  env $1=$V timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$V.log 2>&1
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/bench_$V.log') if l.startswith('{')][-1])
print('$1=$V', d['value'], d['serial']['tokens_per_s'], d['best_serial']['tokens_per_s'], 'tbt', round(d['best_serial']['p50_tbt_s']*1e3,4), round(d['split']['p50_tbt_s']*1e3,4), 'ttft', round(d['best_serial']['p50_ttft_s']*1e3,2))"
done
