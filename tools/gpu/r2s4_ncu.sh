# ncu --set full captures: the bench's roofline kernel (8b-cfg3 decode gate/up, 256 rows) and the 8B prefill
# projections at 4096 tokens (gate/up SwiGLU, Wo/Wd residual epilogues)
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gemm_dsk|gemm_decode" --launch-skip 4 -c 2 \
  -o gpurun_out/roof8b python tools/roofline_capture.py --workload 8b-cfg3 > gpurun_out/roof8b.log 2>&1; echo roof rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc --launch-skip 3 -c 3 \
  -o gpurun_out/pre8b python tools/prefill_capture.py --tokens 4096 > gpurun_out/pre8b.log 2>&1; echo pre rc=$?
ls -la gpurun_out/*.ncu-rep
