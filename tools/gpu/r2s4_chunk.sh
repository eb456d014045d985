# chunked prefill: GPU parity (bit-identical to whole prompts + oracle), property suite incl. chunked cases,
# then configs[2] (8B, 512 requests, U[128,2048]/256, Poisson 128) CB vs mixed vs chunked budgets
mkdir -p gpurun_out
O=gpurun_out/chunk.log
: > $O
timeout 900 python -m pytest tests/test_gpu_model.py -k chunked -x -q -s > gpurun_out/chunk_t1.log 2>&1; echo "chunk parity rc=$?" >> $O; grep -E "chunked prefill|passed|failed|Error" gpurun_out/chunk_t1.log | head >> $O
timeout 900 python -m pytest tests/test_gpu_properties.py -x -q > gpurun_out/chunk_t2.log 2>&1; echo "properties rc=$?" >> $O; tail -3 gpurun_out/chunk_t2.log >> $O
RATES=128 N=512 timeout 1800 python tools/cfg3_sweep.py \
  "policy=continuous_batching;max_batch=256;engine.split=0" \
  "policy=chunked_prefill;max_batch=256;chunk_tokens=1024;engine.split=1;engine.fuse=1" \
  "policy=chunked_prefill;max_batch=256;chunk_tokens=2048;engine.split=1;engine.fuse=1" \
  "policy=chunked_prefill;max_batch=256;chunk_tokens=4096;engine.split=1;engine.fuse=1" \
  "policy=chunked_prefill;max_batch=256;chunk_tokens=8192;engine.split=1;engine.fuse=1" \
  "policy=chunked_prefill;max_batch=256;chunk_tokens=0;tbt_target_ms=30;engine.split=1;engine.fuse=1" \
  "policy=chunked_prefill;max_batch=256;chunk_tokens=0;tbt_target_ms=60;engine.split=1;engine.fuse=1" \
  >> $O 2>&1; echo "sweep rc=$?" >> $O
cat $O
