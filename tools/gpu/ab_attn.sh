mkdir -p gpurun_out
O=gpurun_out/ab.log
: > $O
for F in 0 1; do SW_ATTN_FLAT=$F timeout 200 python tools/attn_ab.py --model LLAMA_1B --layers 2 --batch 64 --prompt 100..1500 --save /tmp/ab1b_$F.npy --oracle $((F*3)) >> $O 2>&1; done
for F in 0 1; do SW_ATTN_FLAT=$F timeout 200 python tools/attn_ab.py --model LLAMA_8B --layers 2 --batch 32 --prompt 1..3000 --save /tmp/ab8b_$F.npy >> $O 2>&1; done
python -c "
import numpy as np
for n in ('1b','8b'):
    a=np.load(f'/tmp/ab{n}_0.npy'); b=np.load(f'/tmp/ab{n}_1.npy')
    rel=np.linalg.norm(a-b,axis=1)/np.linalg.norm(a,axis=1)
    print(n,'flat vs unit: per-row rel max',rel.max(),'argmax agree',(a.argmax(1)==b.argmax(1)).mean())
" >> $O 2>&1
timeout 600 python -m pytest tests -m gpu -x -q >> $O 2>&1
for F in 0 1; do SW_ATTN_FLAT=$F timeout 120 python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512 >> $O 2>&1; done
for F in 0 1; do SW_ATTN_FLAT=$F timeout 200 python tools/step_time.py --model LLAMA_8B --batch 128 --prompt 1024 --steps 20 >> $O 2>&1; done
cat $O | grep -v "^\.\.\." | tail -40
