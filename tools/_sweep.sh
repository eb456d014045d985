python tools/policy_sweep.py "policy=pipelined_splitwiser;P=2;max_batch=32;engine.split=0" \
   "policy=pipelined_splitwiser;P=2;max_batch=32;engine.split=1" \
   "policy=pipelined_splitwiser;P=2;max_batch=32;engine.split=1;engine.decode_sms=48" \
   "policy=pipelined_splitwiser;P=2;max_batch=32;engine.split=1;engine.decode_sms=72" \
   "policy=pipelined_splitwiser;P=2;max_batch=32;engine.split=1;engine.decode_sms=96" \
   "policy=pipelined_splitwiser;P=2;max_batch=32;engine.split=1;engine.decode_sms=120" \
   "policy=pipelined_splitwiser;P=4;max_batch=16;engine.split=1;engine.decode_sms=72" \
   "policy=pipelined_splitwiser;P=4;max_batch=16;engine.split=1;engine.decode_sms=96"
