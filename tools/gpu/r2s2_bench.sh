mkdir -p gpurun_out
make -C paper_2505_03763_b200/csrc -j16 > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
make -C oracle > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
tail -15 gpurun_out/gpu_tests.log
timeout 1500 python bench.py > gpurun_out/bench_cfg3.jsonl 2> gpurun_out/bench_cfg3.err; echo bench rc=$?
tail -3 gpurun_out/bench_cfg3.err; cat gpurun_out/bench_cfg3.jsonl
