mkdir -p gpurun_out
O=gpurun_out/dsk_trace2.log
: > $O
for S in "3072 2048 4 64" "28672 4096 2 256" "4096 4096 1 256"; do SW_DSK_TRACE=1 timeout 120 python tools/dsk_trace.py $S >> $O 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_dsk -s 4 -c 1 -o gpurun_out/dsk_gu256 python tools/dsk_trace.py 28672 4096 2 256 > /dev/null 2>&1
cat $O
