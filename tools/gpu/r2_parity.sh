mkdir -p gpurun_out
make -C paper_2505_03763_b200/csrc -j16 > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
python tools/diag/parity_probe.py > gpurun_out/parity_probe.log 2>&1
SW_PREFILL_TC=0 python tools/diag/parity_probe.py > gpurun_out/parity_probe_tc0.log 2>&1
SW_PREFILL_ROPE_FUSED=0 python tools/diag/parity_probe.py > gpurun_out/parity_probe_rope0.log 2>&1
timeout 900 python -m pytest tests/test_gpu_model.py -m gpu -x -q -s > gpurun_out/r2_gpu_model.log 2>&1; echo rc=$?
for f in parity_probe parity_probe_tc0 parity_probe_rope0; do echo "== $f"; cat gpurun_out/$f.log | grep -v Warn; done
grep -E "rel-L2|passed|failed|Error" gpurun_out/r2_gpu_model.log | head -20
