SW_ATTN_FLAT=0 timeout 120 python tools/attn_ab.py --model LLAMA_1B --layers 2 --batch 64 --prompt 1..1500 --oracle 3 2>&1 | tail -1
SW_ATTN_FLAT=0 timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -1
for i in 1 2; do SW_ATTN_FLAT=0 timeout 120 python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512; done
SW_ATTN_FLAT=0 timeout 200 python tools/step_time.py --model LLAMA_8B --batch 128 --prompt 1024 --steps 20
