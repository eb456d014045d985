mkdir -p gpurun_out
make -C paper_2505_03763_b200/csrc -j16 > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_engine.py tests/test_gpu_properties.py -m gpu -q -x -s > gpurun_out/fuse_tests.log 2>&1; echo tests rc=$?
grep -E "mixed|passed|failed|Error|assert" gpurun_out/fuse_tests.log | head -30
RATES=128 N=512 timeout 1500 python tools/cfg3_sweep.py \
  "policy=continuous_batching;max_batch=256;engine.split=0" \
  "policy=mixed_batching;max_batch=256;engine.split=1;engine.fuse=1;engine.chunk_tokens=2048" \
  "policy=mixed_batching;max_batch=256;engine.split=1;engine.fuse=1;engine.chunk_tokens=4096" \
  "policy=mixed_batching;max_batch=256;engine.split=1;engine.fuse=1;engine.chunk_tokens=8192" \
  > gpurun_out/cfg3_fuse.log 2>&1; echo sweep rc=$?
cat gpurun_out/cfg3_fuse.log | tail -8
