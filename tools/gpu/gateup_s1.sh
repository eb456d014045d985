# Llama-1B decode gate/up with S = 1 (SW_DEC_CTAS=250: 128 CTAs) vs the rule (S = 2: 256 CTAs)
for V in 0 250 0 250; do
  echo "== SW_DEC_CTAS=$V"
  SW_DEC_CTAS=$V timeout 300 python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512 2>&1 | tail -1
  SW_DEC_CTAS=$V timeout 300 python tools/step_time.py --model LLAMA_1B --batch 128 --prompt 512 2>&1 | tail -1
done
