# default bench line (8b-cfg3, now with the chunked arm), then compute-sanitizer racecheck / synccheck on split runs
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r2s4.jsonl 2> gpurun_out/bench_r2s4.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_r2s4.jsonl
for T in racecheck synccheck memcheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_run.py > gpurun_out/san_$T.txt 2>&1; echo "$T rc=$?"; tail -4 gpurun_out/san_$T.txt
done
