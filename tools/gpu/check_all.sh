# GPU parity tests + smoke + default bench (used after kernel changes)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
SW_ATTN_FLAT=1 timeout 200 python tools/attn_ab.py --model LLAMA_8B --layers 2 --batch 32 --prompt 1..3000 --save /tmp/f1.npy > gpurun_out/ab8.log 2>&1
SW_ATTN_FLAT=0 timeout 200 python tools/attn_ab.py --model LLAMA_8B --layers 2 --batch 32 --prompt 1..3000 --save /tmp/f0.npy >> gpurun_out/ab8.log 2>&1
python -c "
import numpy as np
a=np.load('/tmp/f0.npy'); b=np.load('/tmp/f1.npy')
rel=np.linalg.norm(a-b,axis=1)/np.linalg.norm(a,axis=1)
print('8b flat vs unit: per-row rel max',rel.max(),'argmax agree',(a.argmax(1)==b.argmax(1)).mean())" >> gpurun_out/ab8.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -2 gpurun_out/gpu_tests.log; cat gpurun_out/smoke.log | tail -2; tail -1 gpurun_out/ab8.log
python -c "
import json
d=json.loads([l for l in open('gpurun_out/bench.log') if l.startswith('{')][-1])
print({k:d[k] for k in ('value','split_over_serial','split_over_best_serial')}, d['serial']['tokens_per_s'], d['best_serial']['tokens_per_s'], d['roofline_decode_step']['frac'], d['e2e']['value'])"
