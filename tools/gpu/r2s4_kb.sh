mkdir -p gpurun_out
O=gpurun_out/kb.log
: > $O
for rep in 1 2; do for V in base new; do cp abso/libsplitwise_$V.so paper_2505_03763_b200/libsplitwise.so
  for M in "LLAMA_1B --batch 64 --prompt 512" "LLAMA_1B --batch 32 --prompt 2048" "LLAMA_1B --batch 64 --prompt 1024"; do echo "$V $(timeout 300 python tools/step_time.py --model $M --steps 50 2>&1 | tail -1)" >> $O; done; done; done
cp abso/libsplitwise_new.so paper_2505_03763_b200/libsplitwise.so
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -1 >> $O
cat $O
