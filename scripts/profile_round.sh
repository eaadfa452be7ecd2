# One-GPU evidence for the headline config (run under gpurun): bench line,
# launch list of one profiled solve, --set full capture of the top kernels.
# (ncu does not descend into the conditional-node loop graph: the profiled
# solves run the per-iteration graph, PAIRAMG_GRAPH_LOOP=0 -- same kernels.)
# Then: python scripts/ncu_summary.py --launches gpurun_out/launches.csv \
#   --rep gpurun_out/prof_r01.ncu-rep --tag r01 \
#   --key "l1_jacobi_sweep_L0=k_sten2<1, 0, 7" --key "residual_L0=k_sten2<2, 0, 7"
mkdir -p gpurun_out
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/b1.json 2> gpurun_out/b1.err || exit 1
PAIRAMG_GRAPH_LOOP=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches.csv python scripts/profile_solve.py --iters 2 > gpurun_out/ncu_l.log 2>&1 || exit 2
PAIRAMG_GRAPH_LOOP=0 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k 'regex:k_sten2|k_update|k_restrict_c|k_prolong_c4' --launch-count 14 -o gpurun_out/prof_r01 -f \
    python scripts/profile_solve.py --iters 2 > gpurun_out/ncu_f.log 2>&1 || exit 3
echo profile_round ok
