#!/bin/bash
# BASELINE config 4: peak HBM and throughput vs slice count (spatial_k = temporal_k = k).
#   bash tools/slice_sweep.sh > profiles/r02_c4_slice_sweep.txt
echo "# C4 (64f x 4x72x128, base 320, K=25 rehash 13/25), spatial_k = temporal_k = k slices per group"
echo "# k  steps/s  peak_hbm_GB  slice_scratch_GB  arena_GB"
for k in 1 2 4 8 16; do
  python bench.py --config c4 --steps 2 --warmup 3 --no-cpu --no-north-star-plan --spatial-k $k --temporal-k $k 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print($k, d['value'], d['peak_hbm_bytes']/1e9, d['scratch_bytes']/1e9, d['arena_bytes']/1e9)"
done
