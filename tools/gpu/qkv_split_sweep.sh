# decode QKV projection split-K factor sweep (SW_DEC_S_QKV; 0 = the headroom rule)
for V in 0 3 4 5 0 3 4 5; do
  echo "== SW_DEC_S_QKV=$V"
  SW_DEC_S_QKV=$V timeout 300 python tools/step_time.py --model LLAMA_8B --batch 128 --prompt 1024 2>&1 | tail -1
  SW_DEC_S_QKV=$V timeout 300 python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512 2>&1 | tail -1
done
