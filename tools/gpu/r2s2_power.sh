mkdir -p gpurun_out
make -C paper_2505_03763_b200/csrc -j16 > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_engine.py tests/test_gpu_properties.py -m gpu -q -x -s > gpurun_out/fuse_tests.log 2>&1; echo tests rc=$?
grep -E "mixed|passed|failed|Error|assert" gpurun_out/fuse_tests.log | head -30
timeout 600 python tools/power_probe.py --decode-sms 48 > gpurun_out/power_probe.txt 2>&1; echo probe rc=$?
cat gpurun_out/power_probe.txt | grep -v Warn
