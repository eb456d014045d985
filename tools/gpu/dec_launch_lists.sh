# ncu launch lists (gpu time + DRAM bytes per launch) of one decode step in the HBM-bound regime:
# Llama-8B b=64 and b=128 at ctx 1216, Llama-1B b=64 ctx 512 (configs[1]); summarised by tools/ncu_summary.py
mkdir -p gpurun_out/dl
F=gpurun_out/dl
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv"
timeout 600 ncu $M --log-file $F/dec8b_64.csv python tools/profile_step.py --model LLAMA_8B --batch 64 --prompt 1216 --region decode > /dev/null 2>&1
timeout 600 ncu $M --log-file $F/dec8b_128.csv python tools/profile_step.py --model LLAMA_8B --batch 128 --prompt 1216 --region decode > /dev/null 2>&1
timeout 600 ncu $M --log-file $F/dec1b_64.csv python tools/profile_step.py --model LLAMA_1B --batch 64 --prompt 512 --region decode > /dev/null 2>&1
python tools/ncu_summary.py $F/dec8b_64.csv $F/dec8b_128.csv $F/dec1b_64.csv > $F/launch_summary.txt 2>&1
cat $F/launch_summary.txt
