mkdir -p gpurun_out
make -C paper_2505_03763_b200/csrc -j16 > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
nproc; free -g | head -2
timeout 1800 python -m pytest tests/test_gpu_model.py -m gpu -q -s --durations=0 > gpurun_out/r2_gpu_model.log 2>&1; echo rc=$?
grep -E "vs fp32|rel |passed|failed|Error|assert" gpurun_out/r2_gpu_model.log | head -40
grep -E "s call" gpurun_out/r2_gpu_model.log | head -20
