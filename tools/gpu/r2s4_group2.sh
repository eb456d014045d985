mkdir -p gpurun_out
O=gpurun_out/group2.log
: > $O
for rep in 1 2; do for G in 0 16 24 32 48; do
  echo "SW_GEMM_GROUP_MB=$G $(SW_GEMM_GROUP_MB=$G timeout 300 python tools/prefill_time.py --prompts 30 --len 1088 --reps 3 2>&1 | tail -1)" >> $O
done; done
cat $O
