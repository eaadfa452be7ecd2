# A/B of the 27-point level-0 kernels (pencil vs one-row-per-thread): ncu --set full
# of one sweep, residual and SpMV+dots launch of each (development aid, one GPU).
mkdir -p gpurun_out
for v in 1 0; do
  PAIRAMG_STENP=$v PAIRAMG_GRAPH_LOOP=0 timeout 600 ncu --set full --clock-control none --import-source on \
    --profile-from-start off -k 'regex:k_sten' --launch-count 6 -o gpurun_out/ab27_p$v -f \
    python scripts/profile_solve.py --stencil 27 --nd 192 --iters 1 > gpurun_out/ab27_p$v.log 2>&1
done
echo ab27 done
