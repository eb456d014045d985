mkdir -p gpurun_out
O=gpurun_out/persist.log
: > $O
for rep in 1 2; do for P in 1024 2048 4096; do for NL in "8 1088" "30 1088" "16 2048" "4 4096"; do set -- $NL
  echo "PERSIST_MAX=$P $(SW_PREFILL_PERSIST_MAX=$P timeout 300 python tools/prefill_time.py --prompts $1 --len $2 --reps 3 2>&1 | tail -1)" >> $O
done; done; done
cat $O
