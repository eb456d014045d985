mkdir -p gpurun_out
O=gpurun_out/tc_check.log
: > $O
for F in 0 1; do echo "SW_PREFILL_TC=$F" >> $O; SW_PREFILL_TC=$F timeout 120 python tools/attn_ab.py --model LLAMA_1B --layers 2 --batch 8 --prompt 100..700 --save /tmp/p1_$F.npy --oracle 3 >> $O 2>&1; done
python -c "
import numpy as np
a=np.load('/tmp/p1_0.npy'); b=np.load('/tmp/p1_1.npy')
rel=np.linalg.norm(a-b,axis=1)/np.linalg.norm(a,axis=1)
print('1b tc vs mma.sync: per-row rel max',rel.max(),'argmax agree',(a.argmax(1)==b.argmax(1)).mean())
" >> $O 2>&1
cat $O
