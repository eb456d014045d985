for P in 0 1; do SW_PREFILL_TC_PERSIST=$P timeout 120 python tools/attn_ab.py --model LLAMA_1B --layers 2 --batch 8 --prompt 100..700 --save /tmp/q1_$P.npy > /dev/null 2>&1; SW_PREFILL_TC_PERSIST=$P timeout 120 python tools/attn_ab.py --model LLAMA_8B --layers 2 --batch 8 --prompt 100..3000 --save /tmp/q8_$P.npy > /dev/null 2>&1; done
python -c "
import numpy as np
for n in ('1','8'):
    a=np.load(f'/tmp/q{n}_0.npy'); b=np.load(f'/tmp/q{n}_1.npy')
    print(n, 'persistent vs per-item: max abs diff', float(np.abs(a-b).max()), 'identical', bool((a==b).all()))
"
for P in 0 1; do SW_PREFILL_TC_PERSIST=$P timeout 120 python tools/attn_ab.py --model LLAMA_1B --layers 2 --batch 8 --prompt 100..700 --save /tmp/r1_$P.npy > /dev/null 2>&1; done
python -c "
import numpy as np
a=np.load('/tmp/q1_1.npy'); b=np.load('/tmp/r1_1.npy'); c=np.load('/tmp/q1_0.npy'); d=np.load('/tmp/r1_0.npy')
print('run-to-run persistent identical', bool((a==b).all()), 'per-item identical', bool((c==d).all()))
"
