mkdir -p gpurun_out
make -C paper_2505_03763_b200/csrc -j16 > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -m gpu -q -x > gpurun_out/gemm2_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gemm2_tests.log
timeout 600 python tools/gemm_vs_cublas.py --tokens 4096,8192,16384 > gpurun_out/gemm_vs_cublas2.txt 2>&1; cat gpurun_out/gemm_vs_cublas2.txt | grep -v Warn
