"""Real-time replay on one B200 through the batcher: every request completes, shard joins are
complete, latencies are positive, and the joined embeddings match a direct encode."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_replay_world1_completes():
    from paper_2502_00937_b200 import core, policies, workload
    from paper_2502_00937_b200.executor import ImagePathExecutor
    from paper_2502_00937_b200.service import ImagePathService
    import dataclasses
    base = core.get_model_spec("llama3.2-11b")
    spec = dataclasses.replace(base, encoder=dataclasses.replace(base.encoder, layers=2, global_layers=1,
                                                                 out_layers=(1, 2)))
    cfg = workload.GeneratorConfig(model=spec, base_rate=20.0, image_request_fraction=1.0,
                                   images_per_request={1: .5, 2: .3, 3: .2}, seed=5)
    reqs = workload.generate(cfg, 1500.0)
    ex = ImagePathExecutor(spec, seed=0)
    svc = ImagePathService(spec, ex, policies=policies.PolicySet(scheduler=policies.SchedulerKind.FIFO),
                           max_batch={"encode": 4})
    res = svc.replay(reqs)
    assert set(res.latencies_ms) == {r.id for r in reqs}
    assert all(v > 0 for v in res.latencies_ms.values())
    s = res.summary()
    assert s["images"] == sum(len(r.images) for r in reqs) and s["p99_ms"] >= s["p50_ms"] > 0


def test_executor_run_item_spans_match_direct_encode():
    from paper_2502_00937_b200 import core
    from paper_2502_00937_b200.batcher import WorkItem
    from paper_2502_00937_b200.core import StageKind
    from paper_2502_00937_b200.executor import ImagePathExecutor
    import dataclasses
    base = core.get_model_spec("llama3.2-11b")
    spec = dataclasses.replace(base, encoder=dataclasses.replace(base.encoder, layers=1, global_layers=1,
                                                                 out_layers=(1,)))
    rng = np.random.default_rng(0)
    imgs = {7: [rng.integers(0, 256, (400, 700, 3), dtype=np.uint8), rng.integers(0, 256, (600, 300, 3), dtype=np.uint8)],
            9: [rng.integers(0, 256, (560, 560, 3), dtype=np.uint8)]}
    ex = ImagePathExecutor(spec, seed=0)
    items = [WorkItem(seq=0, request_id=7, stage=StageKind.ENCODE, size_tokens=0, tiles=0, enqueue_ms=0,
                      ttft_slo_ms=1, shard_images=(1,)),
             WorkItem(seq=1, request_id=9, stage=StageKind.ENCODE, size_tokens=0, tiles=0, enqueue_ms=0,
                      ttft_slo_ms=1)]
    out = ex.run(items, imgs)
    direct = ex.encode_images([imgs[7][1], imgs[9][0]])
    torch.cuda.synchronize()
    assert out.item_spans == {0: (0, 1), 1: (1, 2)}
    assert torch.equal(out.embeds, direct.embeds)


@pytest.mark.parametrize("model", ["llama3.2-11b", "llava-clip-l14-336", "llava-ov-7b", "internvl-26b"])
def test_projector_matches_torch(model):
    """The LLM-side connector of each family (InternVL: LayerNorm(12800) -> MLP, its LayerNorm as
    mmk_layernorm_bf16) against the same projection in fp32 torch."""
    from paper_2502_00937_b200 import core
    from paper_2502_00937_b200.connector import Projector
    spec = core.get_model_spec(model)
    proj = Projector(spec)
    x = (torch.randn(3000, proj.in_dim, device="cuda") * 0.5).bfloat16()
    got = proj(x).float()
    ref = proj.reference(x)
    rel = ((got - ref).norm() / ref.norm()).item()
    assert got.shape == (3000, 4096) and rel < 1e-2, rel


def test_replay_with_connector_projects_every_shard():
    from paper_2502_00937_b200 import core, workload
    from paper_2502_00937_b200.connector import Projector
    from paper_2502_00937_b200.executor import ImagePathExecutor
    from paper_2502_00937_b200.service import ImagePathService
    import dataclasses
    base = core.get_model_spec("llama3.2-11b")
    spec = dataclasses.replace(base, encoder=dataclasses.replace(base.encoder, layers=1, global_layers=1,
                                                                 out_layers=(1,)))
    cfg = workload.GeneratorConfig(model=spec, base_rate=20.0, image_request_fraction=1.0,
                                   images_per_request={1: .6, 2: .4}, seed=2)
    reqs = workload.generate(cfg, 800.0)
    svc = ImagePathService(spec, ImagePathExecutor(spec, seed=0), connector=Projector(spec))
    svc.replay(reqs)
    torch.cuda.synchronize()
    assert len(svc.projected) == len(reqs)
    for (rid, sid), y in svc.projected.items():
        r = next(r for r in reqs if r.id == rid)
        assert y == (r.total_image_tokens, 4096)
