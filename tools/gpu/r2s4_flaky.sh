mkdir -p gpurun_out
O=gpurun_out/flaky.log
: > $O
for i in 1 2 3 4 5 6; do timeout 600 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | grep -E "^E |passed|failed|Error" | head -12 >> $O; done
timeout 300 python tools/diag/ledger_flake.py 2>&1 | head -3 >> $O
timeout 900 python -m pytest tests/test_gpu_properties.py tests/test_experiment_files.py tests/test_cli.py tests/test_shared_kv.py -m gpu -x -q 2>&1 | tail -2 >> $O
cat $O
