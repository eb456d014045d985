mkdir -p gpurun_out
O=gpurun_out/flat_sweep.log
: > $O
SW_ATTN_FLAT=1 timeout 200 python tools/attn_ab.py --model LLAMA_1B --layers 2 --batch 64 --prompt 100..1500 --oracle 3 >> $O 2>&1
SW_ATTN_FLAT=0 timeout 120 python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512 >> $O 2>&1
for C in 4,6,1 8,4,1 8,6,1 4,6,2; do echo "cfg $C" >> $O; SW_ATTN_FLAT_CFG=$C timeout 120 python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512 >> $O 2>&1; done
SW_ATTN_FLAT=0 timeout 200 python tools/step_time.py --model LLAMA_8B --batch 128 --prompt 1024 --steps 20 >> $O 2>&1
for C in 4,3,1 8,3,1 4,2,2; do echo "cfg $C" >> $O; SW_ATTN_FLAT_CFG=$C timeout 200 python tools/step_time.py --model LLAMA_8B --batch 128 --prompt 1024 --steps 20 >> $O 2>&1; done
SW_ATTN_FLAT_CFG=8,4,1 timeout 300 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:attn_decode_flat -c 1 -o gpurun_out/flat1b python tools/profile_step.py --model LLAMA_1B --batch 64 --prompt 512 > gpurun_out/ncu_flat.log 2>&1
grep -v "^\.\.\." $O | grep -v Traceback | tail -30
