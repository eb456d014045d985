mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_properties.py -x -q > gpurun_out/part.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/part.log
timeout 300 ./paper_2505_03763_b200/split_engine_test > gpurun_out/cpp_entry.log 2>&1; echo "cpp rc=$?"; tail -12 gpurun_out/cpp_entry.log
