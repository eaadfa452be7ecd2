# Multi-GPU evidence (run under gpurun --gpus 4): torchrun parity tests at 2 and
# 4 ranks, weak-scaling bench lines N = 1/2/4 (7- and 27-point, one session),
# 585^3 strong scaling at N = 2/4; LOCAL=1 adds the one-GPU LOCAL 585^3
# iteration test (slow: the reference counts at p = 4 and 8).
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 900 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/${TAG}_pytest_mgpu.log 2>&1; tail -n 3 gpurun_out/${TAG}_pytest_mgpu.log
for n in 1 2 4; do
  timeout 600 python bench.py --gpus $n --steps 5 --warmup 3 --no-pipeline --no-cpu-baseline > gpurun_out/${TAG}_b7_n$n.json 2> gpurun_out/${TAG}_b7_n$n.err
  timeout 600 python bench.py --gpus $n --stencil 27 --steps 5 --warmup 3 --no-pipeline --no-cpu-baseline > gpurun_out/${TAG}_b27_n$n.json 2> gpurun_out/${TAG}_b27_n$n.err
done
for n in 2 4; do
  timeout 900 python bench.py --gpus $n --scaling strong --nd 585 --steps 3 --warmup 3 --no-pipeline > gpurun_out/${TAG}_b585_n$n.json 2> gpurun_out/${TAG}_b585_n$n.err
done
if [ "${LOCAL:-0}" = 1 ]; then
  timeout 1500 python -m pytest tests/test_local_ranks.py -x -q -k 585 > gpurun_out/${TAG}_pytest_l585.log 2>&1; tail -n 3 gpurun_out/${TAG}_pytest_l585.log
fi
echo multi_gpu_round done
