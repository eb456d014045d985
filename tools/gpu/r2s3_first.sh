# round 2 session 3: fresh-container baseline (GPU tests, smoke, default bench)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_cfg3.jsonl 2> gpurun_out/bench_cfg3.err; echo bench rc=$?
tail -3 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench_cfg3.jsonl
