python tools/policy_sweep.py "policy=pipelined_splitwiser;P=2;max_batch=32;engine.split=0" \
   "policy=pipelined_splitwiser;P=2;max_batch=32;engine.split=1" \
   "policy=pipelined_splitwiser;P=2;max_batch=32;engine.split=1;engine.lean_prefill=1" \
   "policy=pipelined_splitwiser;P=4;max_batch=16;engine.split=1" \
   "policy=pipelined_splitwiser;P=4;max_batch=16;engine.split=1;engine.lean_prefill=1" \
   "policy=sequential;max_batch=64;engine.split=0"
export MODEL=LLAMA_8B
export BASE="n=128;input=128..2048;output=256;seed=1;arrival=poisson:64"
python tools/policy_sweep.py "policy=continuous_batching;max_batch=128;engine.split=0" \
   "policy=mixed_batching;max_batch=128;engine.split=1" \
   "policy=mixed_batching;max_batch=128;engine.split=1;engine.lean_prefill=1"
