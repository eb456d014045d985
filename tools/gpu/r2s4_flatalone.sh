mkdir -p gpurun_out
O=gpurun_out/flatalone.log
: > $O
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1 >> $O
for B in "256 1216" "128 1024"; do set -- $B; echo "$(timeout 300 python tools/step_time.py --model LLAMA_8B --batch $1 --prompt $2 --steps 20 2>&1 | tail -1)" >> $O; done
echo "$(timeout 300 python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512 --steps 50 2>&1 | tail -1)" >> $O
RATES=128 N=512 timeout 1200 python tools/cfg3_sweep.py "policy=continuous_batching;max_batch=256;engine.split=0" "policy=mixed_batching;max_batch=256;engine.split=1;engine.prefill_priority=1" "policy=chunked_prefill;max_batch=256;chunk_tokens=8192;engine.split=1;engine.fuse=1" >> $O 2>&1
cat $O
