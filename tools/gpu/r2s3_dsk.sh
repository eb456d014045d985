# stream-K decode GEMM (gemm_decode2.cu): op parity, model parity, then A/B vs the cluster split-K form and cuBLAS
mkdir -p gpurun_out
O=gpurun_out/dsk.log
: > $O
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/dsk_t1.log 2>&1; echo "kernels rc=$?" >> $O; tail -3 gpurun_out/dsk_t1.log >> $O
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_mixed.py -x -q > gpurun_out/dsk_t2.log 2>&1; echo "model rc=$?" >> $O; tail -3 gpurun_out/dsk_t2.log >> $O
for D in 0 1; do echo "SW_GEMM_DSK=$D" >> $O; SW_GEMM_DSK=$D timeout 300 python tools/dec_vs_cublas.py 64 128 256 >> $O 2>&1; done
for D in 0 1; do for M in "LLAMA_8B --batch 256 --prompt 1216" "LLAMA_8B --batch 128 --prompt 1024" "LLAMA_1B --batch 64 --prompt 512"; do
  echo "DSK=$D $(SW_GEMM_DSK=$D timeout 300 python tools/step_time.py --model $M --steps 20 2>&1 | tail -1)" >> $O; done; done
cat $O
