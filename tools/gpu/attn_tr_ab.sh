# decode attention: transposed-product inner loop (SW_ATTN_TR=1) vs the default -- parity, kernel probe, configs[2]
mkdir -p gpurun_out
out=gpurun_out/attn_tr_ab.txt
SW_ATTN_TR=1 timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_kernels.py -x -q > gpurun_out/attn_tr_tests.log 2>&1
echo "SW_ATTN_TR=1 model/kernel parity: rc=$? $(tail -1 gpurun_out/attn_tr_tests.log)" >> $out
for tr in 0 1; do
  echo "== SW_ATTN_TR=$tr" >> $out
  SW_ATTN_TR=$tr timeout 400 python tools/attn_clock_probe.py >> $out 2>&1
  SW_ATTN_TR=$tr timeout 300 python tools/step_time.py --model LLAMA_8B --batch 256 --prompt 1216 --steps 20 >> $out 2>&1
  SW_ATTN_TR=$tr timeout 300 python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512 >> $out 2>&1
  SW_ATTN_TR=$tr RATES=128 REPS=2 timeout 600 python tools/cfg3_sweep.py \
    "policy=continuous_batching;max_batch=256;engine.split=0" \
    "policy=mixed_batching;max_batch=256;engine.split=1;engine.prefill_priority=1" >> $out 2>&1
done
cat $out
