# decode attention ring depth under the power cap: NS = 3 (2 CTAs/SM, default) vs NS = 2 (3 CTAs/SM);
# the kernel probe (cool / power-capped) and configs[2] end to end (serial and split arms)
mkdir -p gpurun_out
for ns in 3 2; do
  echo "== SW_ATTN_STAGES=$ns" >> gpurun_out/attn_stages.txt
  SW_ATTN_STAGES=$ns timeout 400 python tools/attn_clock_probe.py >> gpurun_out/attn_stages.txt 2>&1
  SW_ATTN_STAGES=$ns RATES=128 REPS=2 timeout 600 python tools/cfg3_sweep.py \
    "policy=continuous_batching;max_batch=256;engine.split=0" \
    "policy=mixed_batching;max_batch=256;engine.split=1;engine.prefill_priority=1" >> gpurun_out/attn_stages.txt 2>&1
done
cat gpurun_out/attn_stages.txt
