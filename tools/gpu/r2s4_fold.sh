mkdir -p gpurun_out
O=gpurun_out/fold.log
: > $O
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fold_tests.log 2>&1; echo "gpu tests rc=$?" >> $O; tail -1 gpurun_out/fold_tests.log >> $O; grep -E "^E |FAILED" gpurun_out/fold_tests.log | head -5 >> $O
for rep in 1 2; do for F in 0 1; do for NL in "8 1088" "30 1088" "4 8192"; do set -- $NL
  echo "NORM_FOLD=$F $(SW_PREFILL_NORM_FOLD=$F timeout 300 python tools/prefill_time.py --prompts $1 --len $2 --reps 3 2>&1 | tail -1)" >> $O
done; done; done
cat $O
