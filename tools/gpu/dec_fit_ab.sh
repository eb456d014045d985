# A/B of the co-resident-cluster cap on the decode split-K factor (SW_DEC_FIT)
SW_DEC_LOG=1 timeout 300 python tools/step_time.py --model LLAMA_8B --batch 128 --prompt 1024 --steps 5 --reps 1 2>&1 | grep gemm_decode
SW_DEC_LOG=1 timeout 300 python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512 --steps 5 --reps 1 2>&1 | grep gemm_decode
for V in 0 1 0 1; do
  echo "== SW_DEC_FIT=$V"
  SW_DEC_FIT=$V timeout 300 python tools/step_time.py --model LLAMA_8B --batch 128 --prompt 1024 2>&1 | tail -1
  SW_DEC_FIT=$V timeout 300 python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512 2>&1 | tail -1
done
