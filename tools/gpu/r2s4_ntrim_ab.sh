# A/B of two builds of the library (abso/libsplitwise_{base,new}.so): 8B decode step at several batch sizes
mkdir -p gpurun_out
O=gpurun_out/ntrim_ab.log
: > $O
for rep in 1 2; do for V in base new; do cp abso/libsplitwise_$V.so paper_2505_03763_b200/libsplitwise.so
  for B in 256 200 160 129; do echo "$V $(timeout 300 python tools/step_time.py --model LLAMA_8B --batch $B --prompt 1216 --steps 20 2>&1 | tail -1)" >> $O; done; done; done
cp abso/libsplitwise_new.so paper_2505_03763_b200/libsplitwise.so
cat $O
