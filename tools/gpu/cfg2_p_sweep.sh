# Llama-3.2-1B shape, 64 x 512/128, AllAtZero; PipelinedSplitwiser P in {2,4,8} at matched
# max_batch {32,16,8}: split (concurrent streams) vs serial (the same task stream on one stream, steps merged),
# plus the fastest serial schedule (one 64-request batch)
mkdir -p gpurun_out
timeout 900 python tools/policy_sweep.py \
  "policy=sequential;max_batch=64;engine.split=0" \
  "policy=continuous_batching;max_batch=64;engine.split=0" \
  "policy=pipelined_splitwiser;P=2;max_batch=32;engine.split=0" \
  "policy=pipelined_splitwiser;P=2;max_batch=32;engine.split=1;engine.prefill_priority=1" \
  "policy=pipelined_splitwiser;P=4;max_batch=16;engine.split=0" \
  "policy=pipelined_splitwiser;P=4;max_batch=16;engine.split=1;engine.prefill_priority=1" \
  "policy=pipelined_splitwiser;P=8;max_batch=8;engine.split=0" \
  "policy=pipelined_splitwiser;P=8;max_batch=8;engine.split=1;engine.prefill_priority=1" \
  > gpurun_out/cfg2_p_sweep.txt 2>&1
echo "rc=$?" >> gpurun_out/cfg2_p_sweep.txt
cat gpurun_out/cfg2_p_sweep.txt
