set -x
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $R --master-port 29521 replay.py --duration-s 4 --verify --handoff peer --watchdog-s 240 > gpurun_out/rp_verify_peer.json 2> gpurun_out/rp_verify_peer.err; echo rc=$?
tail -1 gpurun_out/rp_verify_peer.json | head -c 300; echo
timeout 300 $R --master-port 29522 replay.py --duration-s 4 --verify --handoff nccl --watchdog-s 240 > gpurun_out/rp_verify_nccl.json 2> gpurun_out/rp_verify_nccl.err; echo rc=$?
grep -o '"verify".*' gpurun_out/rp_verify_*.json
for h in peer nccl peer nccl; do timeout 300 $R --master-port 29523 replay.py --duration-s 10 --connector --handoff $h --watchdog-s 240 > gpurun_out/rp10_$h.json 2>gpurun_out/rp10_$h.err; tail -1 gpurun_out/rp10_$h.json | head -c 330; echo; done
