mkdir -p gpurun_out
O=gpurun_out/resid.log
: > $O
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1 >> $O
for A in 0 1; do echo "SW_DEC_RESID_ONE=$A" >> $O; SW_DEC_RESID_ONE=$A timeout 300 python tools/dec_vs_cublas.py 64 128 256 2>&1 | grep -E "wo|wd" >> $O; done
for rep in 1 2; do for A in 0 1; do for M in "LLAMA_8B --batch 256 --prompt 1216" "LLAMA_8B --batch 128 --prompt 1024" "LLAMA_8B --batch 64 --prompt 1024" "LLAMA_1B --batch 64 --prompt 512"; do
  echo "RESID_ONE=$A $(SW_DEC_RESID_ONE=$A timeout 300 python tools/step_time.py --model $M --steps 20 2>&1 | tail -1)" >> $O; done; done; done
cat $O
