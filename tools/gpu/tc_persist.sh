mkdir -p gpurun_out
O=gpurun_out/tc_persist.log
: > $O
for F in 0 1; do SW_PREFILL_TC=$F timeout 120 python tools/attn_ab.py --model LLAMA_1B --layers 2 --batch 8 --prompt 100..700 --save /tmp/p1_$F.npy --oracle $F >> $O 2>&1; echo "rc=$?" >> $O; done
for F in 0 1; do SW_PREFILL_TC=$F timeout 200 python tools/attn_ab.py --model LLAMA_8B --layers 2 --batch 8 --prompt 100..3000 --save /tmp/p8_$F.npy >> $O 2>&1; echo "rc=$?" >> $O; done
python -c "
import numpy as np
for n in ('1','8'):
    a=np.load(f'/tmp/p{n}_0.npy'); b=np.load(f'/tmp/p{n}_1.npy')
    rel=np.linalg.norm(a-b,axis=1)/np.linalg.norm(a,axis=1)
    print(n,'tc(persistent) vs mma.sync: per-row rel max',rel.max(),'argmax agree',(a.argmax(1)==b.argmax(1)).mean())
" >> $O 2>&1
for M in "LLAMA_1B --batch 32 --prompt 512" "LLAMA_8B --batch 4 --prompt 8192"; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:attn_prefill -c 1 python tools/profile_step.py --model $M --region prefill 2>&1 | grep -E "duration" >> $O
done
for i in 1 2; do timeout 100 python tools/profile_step.py --model LLAMA_1B --batch 32 --prompt 512 --region prefill >> $O 2>&1; done
cat $O
