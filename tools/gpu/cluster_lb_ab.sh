# decode GEMM cluster scheduling policy (SW_DEC_CLUSTER_LB) x split headroom (SW_DEC_FIT)
for R in 1 2; do
for LB in 0 1; do for F in 8 0; do
  echo "== LB=$LB FIT=$F: $(SW_DEC_CLUSTER_LB=$LB SW_DEC_FIT=$F timeout 300 python tools/step_time.py --model LLAMA_8B --batch 128 --prompt 1024 2>&1 | tail -1) | $(SW_DEC_CLUSTER_LB=$LB SW_DEC_FIT=$F timeout 300 python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512 2>&1 | tail -1)"
done; done; done
