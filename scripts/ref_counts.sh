# Reference iteration counts on the GPU box's host (196 GB, 16 cores): the
# 7-point z-box at p = 2/4/8 concurrently (14 threads, ~150 GB), then 585^3
# at p = 8 and p = 4 one at a time (~130 GB each).  One JSON line per run in
# gpurun_out/ref_counts.jsonl (scripts/ref_counts.py).
mkdir -p gpurun_out
for c in zbox7_p2 zbox7_p4 zbox7_p8; do
  timeout 3000 python scripts/ref_counts.py --only $c >> gpurun_out/ref_counts.jsonl 2>> gpurun_out/ref_counts.err &
done
wait
for c in cube585_p8 cube585_p4; do
  timeout 3000 python scripts/ref_counts.py --only $c >> gpurun_out/ref_counts.jsonl 2>> gpurun_out/ref_counts.err
done
echo ref_counts done
