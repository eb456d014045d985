mkdir -p gpurun_out
O=gpurun_out/group.log
: > $O
for rep in 1 2; do for G in 0 80 110; do
  echo "SW_GEMM_GROUP_MB=$G $(SW_GEMM_GROUP_MB=$G timeout 300 python tools/prefill_time.py --prompts 8 --len 1088 --reps 5 2>&1 | tail -1)" >> $O
  echo "SW_GEMM_GROUP_MB=$G $(SW_GEMM_GROUP_MB=$G timeout 300 python tools/prefill_time.py --prompts 30 --len 1088 --reps 3 2>&1 | tail -1)" >> $O
done; done
for G in 0 80; do SW_GEMM_GROUP_MB=$G timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:gemm_tc --launch-skip 200 -c 8 python tools/prefill_time.py --prompts 30 --len 1088 --reps 1 2>/dev/null | grep -E "gemm_tc" | awk -F'","' '{print $5, $(NF-2), $NF}' | head -24 >> $O; echo "--- G=$G" >> $O; done
cat $O
