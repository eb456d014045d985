# persistent tcgen05 prefill attention: snake / last-tile-first item order (new) vs round robin (old)
mkdir -p gpurun_out
cp abso/new.so paper_2505_03763_b200/libsplitwise.so
bash tools/gpu/tc_persist2.sh
for V in old new; do
  cp abso/$V.so paper_2505_03763_b200/libsplitwise.so
  for P in 0 1; do
    for M in "LLAMA_8B --batch 4 --prompt 8192" "LLAMA_8B --batch 16 --prompt 2048" "LLAMA_1B --batch 32 --prompt 512"; do
      echo "$V persist=$P $M: $(SW_PREFILL_TC_PERSIST=$P timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:attn_prefill -c 2 python tools/profile_step.py --model $M --region prefill 2>&1 | grep -E 'duration' | awk '{print $NF}' | tr '\n' ' ')"
    done
  done
done
cp abso/new.so paper_2505_03763_b200/libsplitwise.so
