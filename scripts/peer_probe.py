"""Development probe (2 GPUs): K9 pack written straight into the LLM-backend GPU's memory over
NVLink (symmetric-memory peer mapping) versus pack into local memory + NCCL send.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/peer_probe.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_00937_b200 import ops  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl")
    rows, d, n_inter = int(os.environ.get("ROWS", "51232")), 1280, 5
    width = d * (1 + n_inter)
    g = torch.Generator(device="cuda").manual_seed(5)
    resid = torch.randn(rows, d, device="cuda", generator=g)
    inter = torch.randn(n_inter, rows, d, device="cuda", generator=g).bfloat16()
    buf = symm.empty(rows * width, dtype=torch.bfloat16, device="cuda")
    hdl = symm.rendezvous(buf, dist.group.WORLD)
    local = torch.empty(rows, width, dtype=torch.bfloat16, device="cuda")
    ref = ops.pack_mllama(resid, inter)
    nbytes = rows * width * 2
    res = {}
    if rank == 1:
        remote = hdl.get_buffer(0, (rows, width), torch.bfloat16)
    modes = os.environ.get("MODES", "nccl,peer,staged,nccl,peer,staged,local,local_staged").split(",")
    for mode in modes:
        buf.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        times = []
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if rank == 1:
                s.record()
                if mode == "peer":
                    ops.pack_mllama(resid, inter, out=remote)
                elif mode == "staged":
                    ops.pack_mllama(resid, inter, out=remote, peer=True)
                elif mode == "local":
                    ops.pack_mllama(resid, inter, out=local)
                elif mode == "local_staged":
                    ops.pack_mllama(resid, inter, out=local, peer=True)
                else:
                    ops.pack_mllama(resid, inter, out=local)
                    dist.send(local, 0)
                e.record()
                torch.cuda.synchronize()
                times.append(s.elapsed_time(e))
            else:
                if mode == "nccl":
                    dist.recv(buf.view(rows, width), 1)
                torch.cuda.synchronize()
            dist.barrier()
        ok = None
        if rank == 0 and not mode.startswith("local"):
            ok = bool(torch.equal(buf.view(rows, width), ref))
        if rank == 1 and mode.startswith("local"):
            ok = bool(torch.equal(local, ref))
        # signal round trip: rank 0 releases, rank 1's stream waits for it
        if rank == 0:
            hdl.put_signal(1, 0)
        else:
            hdl.wait_signal(0, 0, 10000)
        torch.cuda.synchronize()
        t = [torch.tensor([min(times) if times else 0.0, float(ok) if ok is not None else -1.0], device="cuda")]
        dist.all_reduce(t[0], op=dist.ReduceOp.MAX)
        ms = float(t[0][0])
        res.setdefault(mode, []).append({"ms": round(ms, 3), "GB/s": round(nbytes / ms / 1e6, 1),
                                         "bit_exact": bool(t[0][1] > 0)})
    if rank == 0:
        print(json.dumps({"rows": rows, "width": width, "bytes": nbytes, "results": res,
                          "multicast": bool(symm._SymmetricMemory.has_multicast_support(
                              torch._C._autograd.DeviceType.CUDA, 0))}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
