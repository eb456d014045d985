mkdir -p gpurun_out
make -C paper_2505_03763_b200/csrc -j16 > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 600 python tools/gemm_vs_cublas.py --tokens 4096,8192 > gpurun_out/gemm_vs_cublas.txt 2>&1; cat gpurun_out/gemm_vs_cublas.txt | grep -v Warn
