mkdir -p gpurun_out
O=gpurun_out/staged.log
: > $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -3 >> $O
for A in 1 0; do echo "SW_DSK_ALIGNED=$A" >> $O; SW_DSK_ALIGNED=$A timeout 300 python tools/dec_vs_cublas.py 256 2>&1 | grep 8b >> $O; done
SW_DSK_TRACE=1 timeout 120 python tools/dsk_trace.py 6144 4096 4 256 >> $O 2>&1
SW_DSK_TRACE=1 timeout 120 python tools/dsk_trace.py 4096 14336 1 256 >> $O 2>&1
for A in 1 0; do echo "ALIGNED=$A $(SW_DSK_ALIGNED=$A timeout 300 python tools/step_time.py --model LLAMA_8B --batch 256 --prompt 1216 --steps 20 2>&1 | tail -1)" >> $O; done
timeout 1200 python -m pytest tests/test_gpu_model.py -x -q 2>&1 | tail -1 >> $O
cat $O
