# CUPTI kernel timelines (scripts/trace_solve.py) at N = 1 and N = 2 on one
# box (run under gpurun --gpus 2), 7- and 27-point weak problems, on the
# per-iteration graph (CUPTI does not see the conditional-loop graph's kernels).
mkdir -p gpurun_out/trace
export PAIRAMG_GRAPH_LOOP=0
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29555"
for st in 7 27; do
  nd=256; [ $st = 27 ] && nd=192
  timeout 300 python scripts/trace_solve.py --stencil $st --nd $nd --tag n1_$st 2>&1 | tail -1
  timeout 300 $TR scripts/trace_solve.py --stencil $st --nd $nd --tag n2_$st 2>&1 | grep -v "^\*\|OMP" | tail -1
done
timeout 300 $TR scripts/trace_solve.py --stencil 27 --nd 192 --replicate-rows 1000000 --tag n2_27_rep1m 2>&1 | tail -1
echo trace done
