# One-GPU evidence for a round (run under gpurun; TAG=r02 by default):
#  1. the bench line of configs[1] (7-point 256^3),
#  2. the ncu launch list of one profiled 7-point solve (gpu__time_duration,
#     cold-cache and serialised: compare kernel SHARES with the bench),
#  3. ncu --set full of the level-0 kernels: 7-point sweep/residual/dots/update,
#     27-point marching kernels at 192^3, the PLAIN sweep of the varcoef operator.
# (ncu does not descend into the conditional-node loop graph: the profiled
# solves run the per-iteration graph, PAIRAMG_GRAPH_LOOP=0 -- same kernels.)
# Then, here: python scripts/ncu_summary.py --launches gpurun_out/${TAG}_launches.csv \
#   --rep gpurun_out/${TAG}_full7.ncu-rep --tag ${TAG} --key "l1_jacobi_sweep_L0=k_sten2<1, 0, 7"
TAG=${TAG:-r02}
mkdir -p gpurun_out
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench7.json 2> gpurun_out/${TAG}_bench7.err || exit 1
PAIRAMG_GRAPH_LOOP=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/${TAG}_launches.csv python scripts/profile_solve.py --iters 2 > gpurun_out/${TAG}_ncu_l.log 2>&1 || exit 2
PAIRAMG_GRAPH_LOOP=0 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k 'regex:k_sten2|k_update|k_restrict_c|k_prolong_c4' --launch-count 10 -o gpurun_out/${TAG}_full7 -f \
    python scripts/profile_solve.py --iters 2 > gpurun_out/${TAG}_ncu_f7.log 2>&1 || exit 3
PAIRAMG_GRAPH_LOOP=0 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k 'regex:k_sten_march' --launch-count 6 -o gpurun_out/${TAG}_full27 -f \
    python scripts/profile_solve.py --stencil 27 --nd 192 --iters 1 > gpurun_out/${TAG}_ncu_f27.log 2>&1 || exit 4
PAIRAMG_GRAPH_LOOP=0 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k 'regex:k_sell' --launch-count 4 -o gpurun_out/${TAG}_fullplain -f \
    python scripts/profile_solve.py --problem varcoef --levels 0 --format plain --iters 1 > gpurun_out/${TAG}_ncu_fp.log 2>&1 || exit 5
# raw-page CSV exports here; the reports themselves exceed gpurun's 64 MiB copy-back
for r in gpurun_out/${TAG}_full7 gpurun_out/${TAG}_full27 gpurun_out/${TAG}_fullplain; do
  ncu -i $r.ncu-rep --page raw --csv > ${r}_raw.csv 2>/dev/null
  ncu -i $r.ncu-rep --page details --csv > ${r}_details.csv 2>/dev/null
  rm -f $r.ncu-rep
done
echo profile_round ok
