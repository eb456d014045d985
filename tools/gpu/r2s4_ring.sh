mkdir -p gpurun_out
O=gpurun_out/ring.log
: > $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -1 >> $O
timeout 300 python tools/dec_vs_cublas.py 256 2>&1 | grep 8b.gu >> $O
SW_DSK_TRACE=1 timeout 120 python tools/dsk_trace.py 28672 4096 2 256 >> $O 2>&1
echo "$(timeout 300 python tools/step_time.py --model LLAMA_8B --batch 256 --prompt 1216 --steps 20 2>&1 | tail -1)" >> $O
timeout 600 python -m pytest tests/test_gpu_model.py -x -q -k "wide" 2>&1 | tail -1 >> $O
cat $O
