# sweep of the decode split-K GPC headroom (SW_DEC_FIT)
for V in 8 4 12 16 8 4 12 16; do
  echo "== SW_DEC_FIT=$V"
  SW_DEC_FIT=$V SW_DEC_LOG=1 timeout 300 python tools/step_time.py --model LLAMA_8B --batch 128 --prompt 1024 2>&1 | grep -v "K=14336\|mode=2" | tail -3
  SW_DEC_FIT=$V timeout 300 python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512 2>&1 | tail -1
  SW_DEC_FIT=$V timeout 300 python tools/step_time.py --model LLAMA_1B --batch 128 --prompt 512 2>&1 | tail -1
done
