# round-end style validation at HEAD: GPU suite, smoke, default bench line, decode-step / prefill launch lists
mkdir -p gpurun_out/final
F=gpurun_out/final
timeout 2400 python -m pytest tests -m gpu -q > $F/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 $F/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $F/smoke.log
timeout 1200 python bench.py > $F/bench.jsonl 2> $F/bench.err; echo "bench rc=$?"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --profile-from-start off"
timeout 600 ncu $M --log-file $F/dec8b_256.csv python tools/profile_step.py --model LLAMA_8B --batch 256 --prompt 1216 --region decode > /dev/null 2>&1
timeout 600 ncu $M --log-file $F/pre8b_8x1088.csv python tools/profile_step.py --model LLAMA_8B --batch 8 --prompt 1088 --region prefill > /dev/null 2>&1
python tools/ncu_summary.py $F/dec8b_256.csv $F/pre8b_8x1088.csv > $F/launch_summary.txt 2>&1
timeout 300 python tools/step_time.py --model LLAMA_8B --batch 256 --prompt 1216 --steps 20 >> $F/launch_summary.txt 2>&1
cat $F/launch_summary.txt | head -30
python -c "import json;d=json.loads(open('$F/bench.jsonl').read().strip().splitlines()[-1]);print({k:d[k] for k in ('value','split_over_best_serial','roofline')});print(d['chunked']);print(d['serial'])"
