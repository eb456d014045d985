mkdir -p gpurun_out
O=gpurun_out/occ1.log
: > $O
SW_DEC256_OCC1=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -1 >> $O
for A in 0 1; do echo "SW_DEC256_OCC1=$A" >> $O; SW_DEC256_OCC1=$A timeout 300 python tools/dec_vs_cublas.py 256 2>&1 | grep 8b >> $O; done
for S in "6144 4096 4 256" "4096 4096 1 256" "4096 14336 1 256"; do SW_DEC256_OCC1=1 SW_DEC_TRACE=1 timeout 120 python tools/dsk_trace.py $S >> $O 2>&1; done
for A in 0 1; do echo "OCC1=$A $(SW_DEC256_OCC1=$A timeout 300 python tools/step_time.py --model LLAMA_8B --batch 256 --prompt 1216 --steps 20 2>&1 | tail -1)" >> $O; done
SW_DEC256_OCC1=1 timeout 900 python -m pytest tests/test_gpu_model.py -x -q -k "wide" 2>&1 | tail -1 >> $O
cat $O
