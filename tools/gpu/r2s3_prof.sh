# round 2 session 3: where the cfg3 time goes -- decode step b=256 launch list (8B, ctx 1216),
# ncu full of the decode gate/up GEMM and the decode attention at b=256, a cfg3-like prefill launch list
mkdir -p gpurun_out/prof
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --profile-from-start off"
timeout 300 python tools/step_time.py --model LLAMA_8B --batch 256 --prompt 1216 --steps 20 > gpurun_out/prof/step8b_256.txt 2>&1
timeout 300 python tools/step_time.py --model LLAMA_8B --batch 128 --prompt 1024 --steps 20 >> gpurun_out/prof/step8b_256.txt 2>&1
timeout 300 python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512 --steps 50 >> gpurun_out/prof/step8b_256.txt 2>&1
timeout 600 ncu $M --log-file gpurun_out/prof/dec8b_256.csv python tools/profile_step.py --model LLAMA_8B --batch 256 --prompt 1216 --region decode > /dev/null 2>&1
timeout 600 ncu $M --log-file gpurun_out/prof/pre8b_8x1088.csv python tools/profile_step.py --model LLAMA_8B --batch 8 --prompt 1088 --region prefill > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:gemm_decode_kernel -c 4 -o gpurun_out/prof/dec8b_256_gemm python tools/profile_step.py --model LLAMA_8B --batch 256 --prompt 1216 --region decode > gpurun_out/prof/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:attn_decode -c 1 -o gpurun_out/prof/dec8b_256_attn python tools/profile_step.py --model LLAMA_8B --batch 256 --prompt 1216 --region decode > gpurun_out/prof/ncu_attn.log 2>&1
python tools/ncu_summary.py gpurun_out/prof/dec8b_256.csv gpurun_out/prof/pre8b_8x1088.csv
cat gpurun_out/prof/step8b_256.txt
ls -la gpurun_out/prof
