mkdir -p gpurun_out
make -C paper_2505_03763_b200/csrc -j16 > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_model.py tests/test_gpu_kernels.py -m gpu -q -x -s > gpurun_out/b256_tests.log 2>&1; echo tests rc=$?
grep -E "mixed|passed|failed|Error|assert" gpurun_out/b256_tests.log | head -30
timeout 1500 python bench.py > gpurun_out/bench_b256.jsonl 2> gpurun_out/bench_b256.err; echo bench rc=$?
python - <<'PY'
import json; d=json.loads(open("gpurun_out/bench_b256.jsonl").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value","split_over_serial")}, d["serial"], d["roofline"]["achieved"], d["roofline"]["frac"], d["clocks"])
PY
RATES=128 N=512 timeout 1500 python tools/cfg3_sweep.py \
  "policy=mixed_batching;max_batch=256;engine.split=1;engine.decode_sms=48" \
  "policy=mixed_batching;max_batch=256;engine.split=1;engine.decode_sms=64" \
  "policy=mixed_batching;max_batch=256;engine.split=1;engine.decode_sms=96" \
  > gpurun_out/cfg3_smsplit.log 2>&1; echo sweep rc=$?
tail -4 gpurun_out/cfg3_smsplit.log
timeout 300 python tools/power_probe.py --decode-sms 96 > gpurun_out/power_probe_96.txt 2>&1; grep -v Warn gpurun_out/power_probe_96.txt
