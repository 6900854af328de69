for shape in "plain 230400 320 960" "plain 230400 320 320" "plain 230400 320 640" "tconv 25x9216 320 320" "conv 25x72x128 320 320" "conv 25x36x64 1920 640"; do
  for lib in "" variants/nogn.so "" variants/nogn.so; do SF_LIB=${lib:+$PWD/$lib} timeout 60 python tools/gemm_bench.py $shape --reps 50 2>&1 | tail -1 | sed "s|^|${lib:-head} |"; done
done
for lib in "" variants/nogn.so; do SF_LIB=${lib:+$PWD/$lib} timeout 300 python tools/step_once.py --detail --key-only > gpurun_out/det_gn.txt 2>&1; grep sf_gemm gpurun_out/det_gn.txt | awk -v l=${lib:-head} '{s+=$1} END {print l,"key-step gemm sum", s}'; done
