mkdir -p gpurun_out
O=gpurun_out/dsk_trace.log
: > $O
for S in "3072 2048 4 64" "4096 4096 1 64" "28672 4096 2 64" "28672 4096 2 256" "4096 4096 1 256"; do SW_DSK_TRACE=1 timeout 120 python tools/dsk_trace.py $S >> $O 2>&1; done
cat $O
