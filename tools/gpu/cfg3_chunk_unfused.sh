# configs[2]: chunked prefill without fusing the token step (prompt chunks and token steps on two streams,
# prefill priority) and on one stream, beside continuous batching (serial) and mixed batching (split)
mkdir -p gpurun_out
RATES=128 REPS=2 timeout 900 python tools/cfg3_sweep.py \
  "policy=continuous_batching;max_batch=256;engine.split=0" \
  "policy=mixed_batching;max_batch=256;engine.split=1;engine.prefill_priority=1" \
  "policy=chunked_prefill;max_batch=256;chunk_tokens=8192;engine.split=1;engine.fuse=1" \
  "policy=chunked_prefill;max_batch=256;chunk_tokens=8192;engine.split=1;engine.prefill_priority=1" \
  "policy=chunked_prefill;max_batch=256;chunk_tokens=16384;engine.split=1;engine.prefill_priority=1" \
  "policy=chunked_prefill;max_batch=256;chunk_tokens=8192;engine.split=0" > gpurun_out/cfg3_chunk_unfused.txt 2>&1
echo "rc=$?" >> gpurun_out/cfg3_chunk_unfused.txt
cat gpurun_out/cfg3_chunk_unfused.txt
