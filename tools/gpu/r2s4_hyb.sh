# DP + stream-K remainder decode GEMM (gemm_decode2.cu) for projections with more tiles than SMs:
# op parity, A/B vs the cluster form on the 8B gate/up, phase trace, 8B step time
mkdir -p gpurun_out
O=gpurun_out/hyb.log
: > $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/hyb_t1.log 2>&1; echo "kernels rc=$?" >> $O; tail -3 gpurun_out/hyb_t1.log >> $O
for D in 0 1; do echo "SW_GEMM_DSK=$D" >> $O; SW_GEMM_DSK=$D timeout 300 python tools/dec_vs_cublas.py 128 256 2>&1 | grep 8b.gu >> $O; done
SW_DSK_TRACE=1 timeout 120 python tools/dsk_trace.py 28672 4096 2 256 >> $O 2>&1
SW_DSK_TRACE=1 timeout 120 python tools/dsk_trace.py 28672 4096 2 128 >> $O 2>&1
for D in 0 1; do for M in "LLAMA_8B --batch 256 --prompt 1216" "LLAMA_8B --batch 128 --prompt 1024"; do
  echo "DSK=$D $(SW_GEMM_DSK=$D timeout 300 python tools/step_time.py --model $M --steps 20 2>&1 | tail -1)" >> $O; done; done
cat $O
