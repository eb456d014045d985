mkdir -p gpurun_out
RATES=32 N=128 MAXDEC=128 timeout 1500 python tools/cfg3_sweep.py \
  "policy=continuous_batching;max_batch=128;engine.split=0" \
  "policy=mixed_batching;max_batch=128;engine.split=1" \
  "policy=mixed_batching;max_batch=128;engine.split=1;engine.prefill_priority=1" \
  "policy=mixed_batching;max_batch=128;engine.split=1;engine.align=0" \
  "policy=chunked_prefill;max_batch=128;chunk_tokens=8192;engine.split=1;engine.fuse=1" \
  "policy=chunked_prefill;max_batch=128;chunk_tokens=2048;engine.split=1;engine.fuse=1" > gpurun_out/poisson.log 2>&1
cat gpurun_out/poisson.log
