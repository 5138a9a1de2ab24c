# 4-GPU replay: fused pack + NVLink handoff (peer) vs pack + NCCL send, bit-exact check + latency A/B
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $R --master-port 29541 replay.py --duration-s 4 --verify --handoff peer --watchdog-s 240 > gpurun_out/rp4_verify_peer.json 2> gpurun_out/rp4_verify_peer.err; echo rc=$?
grep -o '"handoff".*' gpurun_out/rp4_verify_peer.json
for h in peer nccl peer nccl; do timeout 300 $R --master-port 29542 replay.py --duration-s 10 --connector --handoff $h --watchdog-s 240 > gpurun_out/rp4_10_$h.json 2>gpurun_out/rp4_10_$h.err; tail -1 gpurun_out/rp4_10_$h.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['handoff'], d['handoff_shards'], d['images_per_s'], d['p50_ms'], d['p90_ms'], d['p99_ms'], d['mean_ms'])"; cp gpurun_out/rp4_10_$h.json gpurun_out/rp4_10_${h}_$RANDOM.json; done
