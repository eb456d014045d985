mkdir -p gpurun_out
O=gpurun_out/tc_check2.log
: > $O
for F in 0 1; do SW_PREFILL_TC=$F timeout 200 python tools/attn_ab.py --model LLAMA_8B --layers 2 --batch 8 --prompt 100..3000 --save /tmp/p8_$F.npy >> $O 2>&1; done
python -c "
import numpy as np
a=np.load('/tmp/p8_0.npy'); b=np.load('/tmp/p8_1.npy')
rel=np.linalg.norm(a-b,axis=1)/np.linalg.norm(a,axis=1)
print('8b tc vs mma.sync: per-row rel max',rel.max(),'argmax agree',(a.argmax(1)==b.argmax(1)).mean())
" >> $O 2>&1
for F in 0 1; do for M in "LLAMA_1B --batch 64 --prompt 512" "LLAMA_8B --batch 4 --prompt 8192" "LLAMA_8B --batch 16 --prompt 2048"; do echo "TC=$F $M" >> $O; SW_PREFILL_TC=$F timeout 300 python tools/profile_step.py --model $M --region prefill >> $O 2>&1; SW_PREFILL_TC=$F timeout 300 python tools/profile_step.py --model $M --region prefill >> $O 2>&1; done; done
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --profile-from-start off -k regex:attn_prefill_tc -c 1 python tools/profile_step.py --model LLAMA_1B --batch 64 --prompt 512 --region prefill 2>&1 | grep -E "duration|tensor" >> $O
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --profile-from-start off -k regex:attn_prefill_tc -c 1 python tools/profile_step.py --model LLAMA_8B --batch 4 --prompt 8192 --region prefill 2>&1 | grep -E "duration|tensor" >> $O
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> $O
cat $O
