for shape in "plain 230400 320 960" "plain 230400 320 640" "plain 57600 640 1920"; do
  echo "== $shape (auto)"; python tools/gemm_bench.py $shape --reps 20 2>&1 | tail -n 1
  for bn in 128 160 192 224 256; do for pr in 0 1; do
    echo -n "BN=$bn PAIR=$pr: "; SF_GEMM_BN=$bn SF_GEMM_PAIR=$pr python tools/gemm_bench.py $shape --reps 20 2>&1 | tail -n 1
  done; done
done
echo "== vt 25x9216 320 320 (auto)"; python tools/gemm_bench.py vt 25x9216 320 320 --reps 20 2>&1 | tail -n 1
