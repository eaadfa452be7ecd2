# Two-GPU split-launch diagnostics (run under gpurun --gpus 2): per-level
# storage (PAIRAMG_VERBOSE) and A/B of the split kernels' early PDL trigger
# (PAIRAMG_PDL bit 16) on the 7- and 27-point weak problems.
mkdir -p gpurun_out/diag
for st in 7 27; do
  PAIRAMG_VERBOSE=1 timeout 300 python bench.py --gpus 2 --stencil $st --steps 5 --warmup 3 --no-pipeline --no-cpu-baseline \
    > gpurun_out/diag/v$st.json 2> gpurun_out/diag/v$st.err
  grep "level" gpurun_out/diag/v$st.err | grep rank | head -20
  for pdl in 15 31 15 31; do
    PAIRAMG_PDL=$pdl timeout 300 python bench.py --gpus 2 --stencil $st --steps 5 --warmup 3 --no-pipeline --no-cpu-baseline \
      > gpurun_out/diag/b${st}_pdl${pdl}_$RANDOM.json 2>/dev/null
  done
done
echo diag done
