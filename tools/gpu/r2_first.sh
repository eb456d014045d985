set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
make -C paper_2505_03763_b200/csrc -j16 > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python -m pytest tests/test_gpu_model.py -m gpu -x -q -s > gpurun_out/r2_gpu_model.log 2>&1; echo rc=$?
grep -E "rel-L2|max" gpurun_out/r2_gpu_model.log | head -20
RATES=32,64,128,inf N=512 timeout 1500 python tools/cfg3_sweep.py \
  "policy=continuous_batching;max_batch=256;engine.split=0" \
  "policy=mixed_batching;max_batch=256;engine.split=1" \
  "policy=mixed_batching;max_batch=256;engine.split=1;engine.prefill_priority=1" \
  > gpurun_out/r2_cfg3_sweep.log 2>&1; echo rc=$?
cat gpurun_out/r2_cfg3_sweep.log | tail -30
