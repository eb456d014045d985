mkdir -p gpurun_out
O=gpurun_out/overlap.log
: > $O
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_model.py -k "mixed or chunked" -x -q 2>&1 | tail -1 >> $O
for V in 0 1; do echo "SW_FUSED_OVERLAP=$V" >> $O; SW_FUSED_OVERLAP=$V timeout 400 python tools/fused_step.py --batch 256 --ctx 1216 --chunks 2048,8192 2>&1 | grep -v "through the prefill" >> $O; done
for V in 0 1; do echo "SW_FUSED_OVERLAP=$V (cfg5 shape)" >> $O; SW_FUSED_OVERLAP=$V timeout 600 python tools/fused_step.py --batch 112 --ctx 8448 --chunks 16384 2>&1 | grep -v "through the prefill" >> $O; done
cat $O
