mkdir -p gpurun_out
O=gpurun_out/kvfloor.log
: > $O
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_properties.py -x -q 2>&1 | tail -1 >> $O; done
RATES=128 N=512 timeout 1500 python tools/cfg3_sweep.py \
  "policy=continuous_batching;max_batch=256;engine.split=0" \
  "policy=chunked_prefill;max_batch=256;chunk_tokens=8192;engine.split=1;engine.fuse=1" \
  "policy=chunked_prefill;max_batch=256;chunk_tokens=16384;engine.split=1;engine.fuse=1" \
  "policy=chunked_prefill;max_batch=256;chunk_tokens=24576;engine.split=1;engine.fuse=1" \
  "policy=chunked_prefill;max_batch=256;chunk_tokens=0;tbt_target_ms=150;chunk_max=24576;engine.split=1;engine.fuse=1" \
  >> $O 2>&1
cat $O
