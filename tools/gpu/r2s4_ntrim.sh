mkdir -p gpurun_out
O=gpurun_out/ntrim.log
: > $O
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1 >> $O
for B in 256 200 160 129 96; do echo "$(timeout 300 python tools/step_time.py --model LLAMA_8B --batch $B --prompt 1216 --steps 20 2>&1 | tail -1)" >> $O; done
RATES=128 N=512 timeout 900 python tools/cfg3_sweep.py "policy=continuous_batching;max_batch=256;engine.split=0" "policy=mixed_batching;max_batch=256;engine.split=1;engine.prefill_priority=1" >> $O 2>&1
cat $O
