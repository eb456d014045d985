mkdir -p gpurun_out
O=gpurun_out/long_ctx.log
: > $O
for M in "LLAMA_8B --batch 32 --prompt 4096 --steps 10" "LLAMA_8B --batch 16 --prompt 8192 --steps 10" "LLAMA_1B --batch 32 --prompt 4096 --steps 20" "LLAMA_1B --batch 128 --prompt 512 --steps 20"; do
  echo "== $M" >> $O
  SW_ATTN_FLAT=0 timeout 200 python tools/step_time.py --model $M >> $O 2>&1
  for C in 4,2,2 4,3,1 4,4,2 8,4,1; do echo "cfg $C" >> $O; SW_ATTN_FLAT_CFG=$C timeout 200 python tools/step_time.py --model $M >> $O 2>&1; done
done
grep -v "^\.\.\." $O | grep -v Traceback | tail -40
