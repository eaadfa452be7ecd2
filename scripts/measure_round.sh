mkdir -p gpurun_out/r01m
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/r01m/bench_n1.json 2> gpurun_out/r01m/bench_n1.err
timeout 300 $T --nproc-per-node 2 --master-port 29541 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/r01m/bench_n2.json
timeout 300 $T --nproc-per-node 4 --master-port 29542 bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/r01m/bench_n4.json
timeout 300 $T --nproc-per-node 4 --master-port 29543 bench.py --gpus 4 --steps 3 --warmup 3 --nd 585 --scaling strong --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/r01m/bench_585_n4.json
timeout 300 $T --nproc-per-node 2 --master-port 29544 bench.py --gpus 2 --steps 3 --warmup 3 --nd 585 --scaling strong --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/r01m/bench_585_n2.json
for n in 1 2 4; do timeout 300 $T --nproc-per-node $n --master-port 2955$n bench.py --gpus $n --steps 3 --warmup 3 --stencil 27 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/r01m/bench27_n$n.json; done
for f in gpurun_out/r01m/*.json; do echo "$f: $(python -c "import json,sys; d=json.load(open('$f')); print(d.get('config',{}).get('workload'), d['ms_per_step'], d.get('config',{}).get('iterations'), d.get('config',{}).get('ms_per_iter'), d.get('e2e',{}).get('value'), (d.get('roofline') or {}).get('frac'))" 2>&1 | tail -1)"; done
