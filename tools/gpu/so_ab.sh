# A/B two builds of libsplitwise.so on one box: bash tools/gpu/so_ab.sh  (abso/old.so vs abso/new.so;
# build each with `make -C paper_2505_03763_b200/csrc` and copy ../libsplitwise.so into abso/, git-ignored)
mkdir -p gpurun_out
for V in old new old new; do
  cp abso/$V.so paper_2505_03763_b200/libsplitwise.so
  echo "== $V"
  timeout 300 python tools/step_time.py --model LLAMA_1B --batch 64 --prompt 512 2>&1 | tail -1
  timeout 300 python tools/step_time.py --model LLAMA_8B --batch 128 --prompt 1024 2>&1 | tail -1
done
cp abso/new.so paper_2505_03763_b200/libsplitwise.so
