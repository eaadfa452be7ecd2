# Extra ncu captures (raw/details CSV exported on the box): the 7-point
# level-0 SpMV+dots kernel and the CODED sweep of the varcoef operator.
TAG=${TAG:-r02}
mkdir -p gpurun_out
PAIRAMG_GRAPH_LOOP=0 timeout 600 ncu --set full --clock-control none --profile-from-start off \
    -k 'regex:k_sten2_dots' --launch-count 1 -o gpurun_out/${TAG}_dots7 -f \
    python scripts/profile_solve.py --iters 1 > gpurun_out/${TAG}_ncu_dots7.log 2>&1
PAIRAMG_GRAPH_LOOP=0 timeout 600 ncu --set full --clock-control none --profile-from-start off \
    -k 'regex:k_sell' --launch-count 4 -o gpurun_out/${TAG}_fullcoded -f \
    python scripts/profile_solve.py --problem varcoef --levels 2 --format coded --iters 1 > gpurun_out/${TAG}_ncu_fc.log 2>&1
for r in gpurun_out/${TAG}_dots7 gpurun_out/${TAG}_fullcoded; do
  ncu -i $r.ncu-rep --page raw --csv > ${r}_raw.csv 2>/dev/null
  ncu -i $r.ncu-rep --page details --csv > ${r}_details.csv 2>/dev/null
  rm -f $r.ncu-rep
done
echo profile_extra ok
