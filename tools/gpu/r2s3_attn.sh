# new warp-specialised tcgen05 prefill attention: parity first, then old vs new kernel time
mkdir -p gpurun_out
O=gpurun_out/attn_new.log
: > $O
cp abso/new.so paper_2505_03763_b200/libsplitwise.so
timeout 120 python tools/attn_ab.py --model LLAMA_1B --layers 2 --batch 8 --prompt 100..700 --save /tmp/p1_1.npy --oracle 1 >> $O 2>&1; echo "rc=$?" >> $O
SW_PREFILL_TC=0 timeout 120 python tools/attn_ab.py --model LLAMA_1B --layers 2 --batch 8 --prompt 100..700 --save /tmp/p1_0.npy >> $O 2>&1
timeout 200 python tools/attn_ab.py --model LLAMA_8B --layers 2 --batch 8 --prompt 100..3000 --save /tmp/p8_1.npy >> $O 2>&1; echo "rc=$?" >> $O
SW_PREFILL_TC=0 timeout 200 python tools/attn_ab.py --model LLAMA_8B --layers 2 --batch 8 --prompt 100..3000 --save /tmp/p8_0.npy >> $O 2>&1
python -c "
import numpy as np
for n in ('1','8'):
    a=np.load(f'/tmp/p{n}_0.npy'); b=np.load(f'/tmp/p{n}_1.npy')
    rel=np.linalg.norm(a-b,axis=1)/np.linalg.norm(a,axis=1)
    print(n,'new tc vs mma.sync: per-row rel max',rel.max(),'argmax agree',(a.argmax(1)==b.argmax(1)).mean())
" >> $O 2>&1
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_kernels.py tests/test_gpu_mixed.py -x -q > gpurun_out/t_attn.log 2>&1; tail -3 gpurun_out/t_attn.log >> $O
for V in old new; do
  cp abso/$V.so paper_2505_03763_b200/libsplitwise.so
  for M in "LLAMA_8B --batch 4 --prompt 8192" "LLAMA_8B --batch 8 --prompt 1088" "LLAMA_1B --batch 32 --prompt 512"; do
    echo "$V $M: $(timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --profile-from-start off -k regex:attn_prefill -c 2 python tools/profile_step.py --model $M --region prefill 2>&1 | grep -E 'duration|tensor' | awk '{print $1, $NF}' | tr '\n' ' ')" >> $O
  done
done
cp abso/new.so paper_2505_03763_b200/libsplitwise.so
cat $O
