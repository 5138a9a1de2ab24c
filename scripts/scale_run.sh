#!/bin/bash
# Multi-GPU bench lines on one box (weak and strong scaling) + the 2-GPU tests.
# Usage: bash scripts/scale_run.sh N   -> gpurun_out/scale_r02_{weak,strong}_n{1..N}.json
set -u
cd "$(dirname "$0")/.."
N=${1:-2}
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r02_gpu_multi_n$N.log 2>&1; tail -2 gpurun_out/r02_gpu_multi_n$N.log
for mode in weak strong; do
  for n in $(seq 1 $N); do
    if [ $n -eq 1 ]; then
      timeout 600 python bench.py --scaling $mode --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/scale_r02_${mode}_n1.json 2>gpurun_out/scale_r02_${mode}_n1.err
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + n)) \
        bench.py --gpus $n --scaling $mode --steps 10 --warmup 3 > gpurun_out/scale_r02_${mode}_n$n.json 2>gpurun_out/scale_r02_${mode}_n$n.err
    fi
    python -c "import json,sys; d=json.loads(open('gpurun_out/scale_r02_${mode}_n$n.json').read().strip().splitlines()[-1]); print('$mode', d['n_gpus'], d['value'], d['ms_per_step'], d['config']['parallelism'], d['clocks'])" 2>&1 | tail -1
  done
done
