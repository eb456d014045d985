# round 2, session 2: state check at HEAD + HBM-per-SM scaling + cfg3 sweep
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; free -g | head -2
make -C paper_2505_03763_b200/csrc -j16 > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
make -C oracle > /dev/null 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/hbm_sm_scaling.cu -o /tmp/hbm_sm && timeout 300 /tmp/hbm_sm > gpurun_out/hbm_sm_scaling.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
tail -25 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
RATES=64,inf N=512 timeout 1500 python tools/cfg3_sweep.py \
  "policy=continuous_batching;max_batch=256;engine.split=0" \
  "policy=mixed_batching;max_batch=256;engine.split=1" \
  "policy=mixed_batching;max_batch=256;engine.split=1;engine.prefill_priority=1" \
  > gpurun_out/cfg3_sweep.log 2>&1; echo sweep rc=$?
cat gpurun_out/cfg3_sweep.log | tail -12
cat gpurun_out/hbm_sm_scaling.txt
