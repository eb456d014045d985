for V in 0 240 0 240 264; do
  echo "== SW_DEC_CTAS=$V"
  SW_DEC_CTAS=$V timeout 300 python tools/step_time.py --model LLAMA_8B --batch 128 --prompt 1024 2>&1 | tail -1
done
SW_DEC_CTAS=240 timeout 300 python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512 2>&1 | tail -1
SW_DEC_CTAS=0 timeout 300 python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512 2>&1 | tail -1
