"""Two-GPU handoff (runs only where the box has >= 2 GPUs; the single-GPU suite skips it).

The replay service with the fused pack + NVLink handoff (PeerShardChannel: encoders on rank 1 pack
straight into rank 0's memory) and with the NCCL payload path; rank 0 re-encodes every remote
shard and compares it bit for bit with what arrived (replay.py --verify)."""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("handoff,port,model,slot_images", [
    ("peer", 29531, "llama3.2-11b", 16), ("nccl", 29532, "llama3.2-11b", 16),
    ("peer", 29533, "llava-clip-l14-336", 16),
    ("peer", 29534, "llama3.2-11b", 1)])  # one-image slots: most batches take the NCCL fallback
def test_replay_handoff_bit_exact(handoff, port, model, slot_images):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "replay.py"),
           "--duration-s", "3", "--verify", "--handoff", handoff, "--model", model, "--slot-images", str(slot_images), "--watchdog-s", "240"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["handoff"] == handoff
    assert line["verify"]["remote_shards"] > 0 and line["verify"]["mismatches"] == 0, line["verify"]
    if handoff == "peer":
        assert line["handoff_shards"]["peer"] > 0
    if slot_images == 1:
        assert line["handoff_shards"]["nccl"] > 0


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("scaling,port", [("weak", 29541), ("strong", 29542)])
def test_bench_two_gpus_json_line(scaling, port):
    """bench.py under torchrun at N=2 (the driver's scaling launch): one JSON line from rank 0 with
    n_gpus 2, the whole-job value, the partition and the NVLink handoff inside the timed region."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--scaling", scaling, "--model", "vit-b16-224"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["parallelism"].startswith("dp2") and "cpu_baseline" not in d
    assert d["config"]["images_per_step"] == (16 if scaling == "weak" else 32)
