"""bench.py's reference arm runs on CPU: its JSON line keeps the driver's contract (one line on
stdout, the metric/unit of the GPU arm, impl=reference, cpu_baseline and e2e objects)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--model", "vit-b16-224",
                        "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "images/sec (preprocess+encode)"
    assert d["unit"] == "images/s" and d["higher_is_better"] is True and d["n_gpus"] == 1
    assert d["steps"] == 1 and d["warmup"] == 3 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "workload" in d["config"]
    # same config as the GPU arm (its batch's tile histogram) and no product CUDA code mapped
    assert d["cpu_baseline"]["same_config"] is True and d["cpu_baseline"]["tile_histogram"] == {"1": 8}
    assert not any("libmmk" in so for so in d["native_so_loaded"])


def test_mix_sampler_weights_the_batch_histogram():
    """The CPU legs' batch-time estimate: per-tile-count mean seconds x the batch's tile counts,
    unsampled tile counts scaled by encoder FLOPs."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2502_00937_b200 import core
    spec = core.get_model_spec("llama3.2-11b")
    dims = bench.image_dims(spec, 32)
    ms = bench.MixSampler(spec, dims, 1000)
    assert sum(ms.hist.values()) == 32 and ms.group == 1
    seen = []
    for _ in range(len(ms.hist)):
        t, imgs = ms.next_sample()
        assert all(core.tile_count(im.shape[1], im.shape[0], spec) == t for im in imgs)
        seen.append(t)
        ms.record(t, 2.0 * t)
    assert sorted(seen) == sorted(ms.hist)
    total, est = ms.batch_seconds()
    assert abs(total - sum(c * 2.0 * t for t, c in ms.hist.items())) < 1e-9
    ms2 = bench.MixSampler(spec, dims, 1000)
    t, _ = ms2.next_sample()
    ms2.record(t, 5.0)
    total2, est2 = ms2.batch_seconds()
    for u in ms2.hist:
        assert abs(est2[u] - 5.0 * bench.encoder_flops(spec, [u]) / bench.encoder_flops(spec, [t])) < 1e-9


import pytest  # noqa: E402


@pytest.mark.gpu
def test_gpu_arm_json_line():
    """The GPU arm's line carries every key the driver and the judge read."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--model", "vit-b16-224", "--steps", "3",
                        "--warmup", "3"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["steps"] == 3 and d["warmup"] == 3
    assert set(d["roofline"]) >= {"bound", "achieved", "peak", "unit", "frac", "traffic"}
    assert 0 < d["roofline"]["frac"] <= 1.5
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
