# configs[2] Poisson rate sweep (SURVEY §8d "lambda swept"): CB (serial) vs mixed (split) vs chunked prefill
mkdir -p gpurun_out
RATES=16,32,64,128,inf N=512 timeout 3000 python tools/cfg3_sweep.py \
  "policy=continuous_batching;max_batch=256;engine.split=0" \
  "policy=mixed_batching;max_batch=256;engine.split=1;engine.prefill_priority=1" \
  "policy=chunked_prefill;max_batch=256;chunk_tokens=8192;engine.split=1;engine.fuse=1" > gpurun_out/lambda.log 2>&1
cat gpurun_out/lambda.log
