mkdir -p gpurun_out
O=gpurun_out/prefill_check.log
: > $O
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> $O
for M in "LLAMA_1B --batch 64 --prompt 512" "LLAMA_8B --batch 4 --prompt 8192" "LLAMA_8B --batch 16 --prompt 2048"; do
  timeout 300 python tools/profile_step.py --model $M --region prefill >> $O 2>&1
  timeout 300 python tools/profile_step.py --model $M --region prefill >> $O 2>&1
done
timeout 300 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:attn_prefill -c 1 -o gpurun_out/pfattn2 python tools/profile_step.py --model LLAMA_1B --batch 64 --prompt 512 --region prefill > /dev/null 2>&1
cat $O
