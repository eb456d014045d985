# C++ entry test + kernel-level partition concurrency (8B and 1B)
mkdir -p gpurun_out
make -C paper_2505_03763_b200/csrc -j16 > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 600 ./paper_2505_03763_b200/split_engine_test > gpurun_out/cpp_entry.log 2>&1; echo cpp rc=$?; tail -20 gpurun_out/cpp_entry.log
timeout 600 python tools/partition_overlap.py --model LLAMA_8B --batch 64 --ctx 1024 --prompts 8 --prompt-len 1024 --decode-sms 24,32,40,48,64,80,96 > gpurun_out/part_8b_b64.txt 2>&1
timeout 600 python tools/partition_overlap.py --model LLAMA_8B --batch 128 --ctx 1024 --prompts 8 --prompt-len 1024 --decode-sms 32,48,64,80 > gpurun_out/part_8b_b128.txt 2>&1
timeout 600 python tools/partition_overlap.py --model LLAMA_1B --batch 64 --ctx 512 --prompts 32 --prompt-len 512 --decode-sms 32,48,64,80 > gpurun_out/part_1b_b64.txt 2>&1
cat gpurun_out/part_*.txt | grep -v Warn
