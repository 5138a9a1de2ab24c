#!/bin/bash
# Multi-GPU evidence on one box: weak-scaling bench lines N=1..N and the replay service (bursty trace
# through route_image / form_batch, routing on the measured profile, fused NVLink handoff, connector,
# every remote shard verified) at N=1, 2, N.   Usage: [SKIP_BENCH=1] bash scripts/multi_run.sh N
set -u
cd "$(dirname "$0")/.."
N=${1:-4}
O=gpurun_out
for n in $(seq 1 $N); do
  [ -n "${SKIP_BENCH:-}" ] && break
  if [ $n -eq 1 ]; then
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/scale_r02b_weak_n1.json 2>$O/scale_r02b_weak_n1.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + n)) \
      bench.py --gpus $n --steps 10 --warmup 3 > $O/scale_r02b_weak_n$n.json 2>$O/scale_r02b_weak_n$n.err
  fi
  python -c "import json; d=json.loads(open('$O/scale_r02b_weak_n$n.json').read().strip().splitlines()[-1]); print('weak', d['n_gpus'], d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
for n in 1 2 $N; do
  if [ $n -eq 1 ]; then
    timeout 600 python replay.py --duration-s 10 --connector > $O/r02_replay_n1.json 2>$O/r02_replay_n1.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700 + n)) \
      replay.py --duration-s 10 --connector --verify --watchdog-s 600 > $O/r02_replay_n$n.json 2>$O/r02_replay_n$n.err
  fi
  tail -c 700 $O/r02_replay_n$n.json; echo
done
