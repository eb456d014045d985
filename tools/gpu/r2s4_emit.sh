mkdir -p gpurun_out
O=gpurun_out/emit.log
: > $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -1 >> $O
timeout 300 python tools/dec_vs_cublas.py 64 128 256 2>&1 >> $O
for M in "LLAMA_8B --batch 256 --prompt 1216" "LLAMA_8B --batch 128 --prompt 1024" "LLAMA_1B --batch 64 --prompt 512"; do
  echo "$(timeout 300 python tools/step_time.py --model $M --steps 20 2>&1 | tail -1)" >> $O; done
timeout 1200 python -m pytest tests/test_gpu_model.py tests/test_gpu_mixed.py -x -q 2>&1 | tail -1 >> $O
cat $O
