# what do the two phases contend for on disjoint SM partitions?
mkdir -p gpurun_out
make -C paper_2505_03763_b200/csrc -j16 > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
A="--model LLAMA_8B --batch 64 --ctx 1024 --prompts 8 --prompt-len 1024 --decode-sms 32,48,64"
echo "## decode = pure read stream of 4 GB (torch sum)" > gpurun_out/interf.txt
timeout 600 python tools/partition_overlap.py $A --stream-gb 4 2>&1 | grep -v Warn >> gpurun_out/interf.txt
echo "## decode = attention only (SW_ABLATE=62)" >> gpurun_out/interf.txt
SW_ABLATE=62 timeout 600 python tools/partition_overlap.py $A 2>&1 | grep -v Warn >> gpurun_out/interf.txt
echo "## decode = GEMMs only (SW_ABLATE=1)" >> gpurun_out/interf.txt
SW_ABLATE=1 timeout 600 python tools/partition_overlap.py $A 2>&1 | grep -v Warn >> gpurun_out/interf.txt
echo "## decode = GEMMs only, b=32 (BN 32: activation re-reads 1.25x of weights)" >> gpurun_out/interf.txt
SW_ABLATE=1 timeout 600 python tools/partition_overlap.py --model LLAMA_8B --batch 32 --ctx 1024 --prompts 8 --prompt-len 1024 --decode-sms 32,48,64 2>&1 | grep -v Warn >> gpurun_out/interf.txt
cat gpurun_out/interf.txt
