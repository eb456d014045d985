mkdir -p gpurun_out
O=gpurun_out/flat_full.log
: > $O
for F in 0 1; do SW_ATTN_FLAT=$F timeout 200 python tools/attn_ab.py --model LLAMA_1B --layers 2 --batch 64 --prompt 1..1500 --save /tmp/a1_$F.npy --oracle $((F*3)) >> $O 2>&1; done
for F in 0 1; do SW_ATTN_FLAT=$F timeout 200 python tools/attn_ab.py --model LLAMA_8B --layers 2 --batch 32 --prompt 1..3000 --save /tmp/a8_$F.npy >> $O 2>&1; done
python -c "
import numpy as np
for n in ('1','8'):
    a=np.load(f'/tmp/a{n}_0.npy'); b=np.load(f'/tmp/a{n}_1.npy')
    rel=np.linalg.norm(a-b,axis=1)/np.linalg.norm(a,axis=1)
    print(n,'flat vs unit: per-row rel max',rel.max(),'argmax agree',(a.argmax(1)==b.argmax(1)).mean())
" >> $O 2>&1
SW_ATTN_FLAT=1 timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t_flat1.log 2>&1; tail -2 gpurun_out/t_flat1.log >> $O
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t_auto.log 2>&1; tail -2 gpurun_out/t_auto.log >> $O
for M in "LLAMA_1B --batch 64 --prompt 512" "LLAMA_1B --batch 32 --prompt 4096 --steps 20" "LLAMA_8B --batch 128 --prompt 1024 --steps 20" "LLAMA_8B --batch 16 --prompt 8192 --steps 10"; do
  for F in 0 1 2; do SW_ATTN_FLAT=$F timeout 200 python tools/step_time.py --model $M >> $O 2>&1; done
done
cat $O | grep -v "^\.\.\." | grep -v Traceback
bash tools/gpu/bench_ab.sh SW_ATTN_FLAT 0 2
