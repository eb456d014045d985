mkdir -p gpurun_out
O=gpurun_out/rope_check.log
: > $O
for F in 0 1; do SW_PREFILL_ROPE_FUSED=$F timeout 120 python tools/attn_ab.py --model LLAMA_1B --layers 2 --batch 8 --prompt 100..700 --save /tmp/r1_$F.npy --oracle $F >> $O 2>&1; done
for F in 0 1; do SW_PREFILL_ROPE_FUSED=$F timeout 200 python tools/attn_ab.py --model LLAMA_8B --layers 2 --batch 8 --prompt 100..3000 --save /tmp/r8_$F.npy >> $O 2>&1; done
python -c "
import numpy as np
for n in ('1','8'):
    a=np.load(f'/tmp/r{n}_0.npy'); b=np.load(f'/tmp/r{n}_1.npy')
    rel=np.linalg.norm(a-b,axis=1)/np.linalg.norm(a,axis=1)
    print(n,'fused vs rope_kv: per-row rel max',rel.max(),'exact rows',(rel==0).mean(),'argmax agree',(a.argmax(1)==b.argmax(1)).mean())
" >> $O 2>&1
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -1 >> $O
for F in 0 1; do for i in 1 2; do SW_PREFILL_ROPE_FUSED=$F timeout 100 python tools/profile_step.py --model LLAMA_1B --batch 32 --prompt 512 --region prefill >> $O 2>&1; done; done
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --profile-from-start off -k regex:gemm_tc_kernel -c 1 python tools/profile_step.py --model LLAMA_1B --batch 32 --prompt 512 --region prefill 2>&1 | grep -E "duration|tensor" >> $O
cat $O
