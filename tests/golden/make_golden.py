"""Generate golden vectors for the image path by running the REFERENCE implementation.

Run in the authoring container (the reference is mounted read-only at /root/reference and is
not available on the GPU box; the JSON outputs are committed instead):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (tests/golden/):
  tiling.json      tile_count / image_tokens for every reference preset over edge-case dims and
                   ~8k generator-drawn dims (reference core.py:58-74)
  generator.json   reference workload.generate() request streams for several seeds/configs
                   (workload.py:222-296)
  profile_llama.json  the reference's calibrated LatencyProfile for llama3.2-11b (export base)
  policies.json    split_by_tiles (policies.py:91-101), route_image (:104-124),
                   schedule_order (:153-173) and form_batch (engine.py:100-114) cases
"""

from __future__ import annotations

import json
import random
from pathlib import Path
from types import SimpleNamespace

from lmmsim import core as rcore
from lmmsim import engine as rengine
from lmmsim import policies as rpol
from lmmsim import workload as rwork

OUT = Path(__file__).resolve().parent


def tiling():
    specs = rcore.load_model_specs()
    dims = [(1, 1), (1, 4096), (4096, 1), (0, 10), (10, 0), (-3, 5), (8000, 8000), (2 ** 31 - 1, 1)]
    for spec in specs.values():
        t = spec.tile_edge_px
        for a in (t - 1, t, t + 1, 2 * t - 1, 2 * t, 2 * t + 1, 3 * t, 4 * t + 1, 5 * t + 7):
            for b in (1, t - 1, t, t + 1, 2 * t + 1):
                dims.append((a, b))
                dims.append((b, a))
    for extra in (224, 336):  # the two single-tile encoder configs of BASELINE.json
        for a in (extra - 1, extra, extra + 1, 2 * extra + 3):
            dims.append((a, extra))
    cfg = rwork.GeneratorConfig(model=specs["llama3.2-11b"], base_rate=50.0, image_request_fraction=1.0, seed=0)
    reqs = rwork.generate(cfg, 25_000.0)
    dims += [(i.width_px, i.height_px) for r in reqs for i in r.images]
    toy = rcore.ModelSpec(name="toy", architecture=rcore.Architecture.DEC_ONLY, tile_edge_px=100,
                          tokens_per_tile=10, max_tiles_per_image=3)
    custom = {
        "vit-b16-224": rcore.ModelSpec("vit-b16-224", rcore.Architecture.DEC_ONLY, 224, 197, 1),
        "llava-clip-l14-336": rcore.ModelSpec("llava-clip-l14-336", rcore.Architecture.DEC_ONLY, 336, 576, 1),
        "toy": toy,
    }
    allspecs = dict(specs)
    allspecs.update(custom)
    out = {}
    for name, spec in allspecs.items():
        rows = []
        for w, h in dims:
            try:
                rows.append([w, h, rcore.tile_count(w, h, spec), rcore.image_tokens(w, h, spec)])
            except rcore.SpecError:
                rows.append([w, h, -1, -1])
        out[name] = {"spec": [spec.tile_edge_px, spec.tokens_per_tile, spec.max_tiles_per_image,
                              int(spec.thumbnail_tile)], "rows": rows}
    (OUT / "tiling.json").write_text(json.dumps(out, separators=(",", ":")))


def generator():
    specs = rcore.load_model_specs()
    cases = []
    for seed, model, kw, horizon in [
        (0, "llama3.2-11b", {}, 120_000.0),
        (7, "llama3.2-11b", {"base_rate": 20.0, "image_request_fraction": 0.9}, 30_000.0),
        (3, "internvl-26b", {"image_dim_median_px": 430.0, "image_dim_sigma": 0.45,
                             "images_per_request": {1: 0.5, 2: 0.3, 3: 0.1, 4: 0.1}}, 60_000.0),
        (11, "llama3.2-11b", {"base_rate": 10.0,
                              "images_per_request": {1: .3, 2: .2, 3: .15, 4: .1, 5: .1, 6: .05, 7: .05, 8: .05},
                              "burst": [[10_000.0, 5_000.0, 3.0, 2.0]]}, 40_000.0),
    ]:
        kw = dict(kw)
        bursts = tuple(rwork.BurstEpisode(*b) for b in kw.pop("burst", []))
        cfg = rwork.GeneratorConfig(model=specs[model], seed=seed, burst_episodes=bursts, **kw)
        reqs = rwork.generate(cfg, horizon)
        cases.append({
            "seed": seed, "model": model, "kw": {k: (v if not isinstance(v, dict) else {str(a): b for a, b in v.items()})
                                                  for k, v in kw.items()},
            "burst": [[b.start_ms, b.duration_ms, b.rate_multiplier, b.image_multiplier] for b in bursts],
            "horizon_ms": horizon,
            "requests": [[r.arrival_ms, r.text_tokens, r.output_tokens, r.service_id,
                          [[i.width_px, i.height_px, i.tiles, i.image_tokens] for i in r.images],
                          r.total_image_tokens, r.total_tiles] for r in reqs],
        })
    (OUT / "generator.json").write_text(json.dumps(cases, separators=(",", ":")))


def policies():
    rnd = random.Random(1234)
    split = [[[5, 4, 3, 3, 1], 2]]
    for _ in range(300):
        tiles = [rnd.randint(1, 10) for _ in range(rnd.randint(1, 16))]
        split.append([tiles, rnd.randint(1, 9)])
    split_out = [[t, n, rpol.split_by_tiles(t, n)] for t, n in split]

    spec = rcore.get_model_spec("llama3.2-11b")
    routes = []
    for case in range(200):
        n_img = rnd.randint(1, 12)
        imgs = tuple(rcore.ImageSpec.from_dims(rnd.randint(64, 2400), rnd.randint(64, 2400), spec) for _ in range(n_img))
        req = rcore.Request(id=case, arrival_ms=0.0, text_tokens=10, images=imgs, output_tokens=1)
        n_inst = rnd.randint(1, 10)
        pend = [rnd.choice([0, 1601, 3202, 6404, rnd.randint(0, 20000)]) for _ in range(n_inst)]
        insts = [SimpleNamespace(id=k, pending_image_tokens=pend[k], pending_text_tokens=0) for k in range(n_inst)]
        router = rnd.choice(list(rpol.RouterKind))
        fan = rnd.randint(1, 9)
        rr = {"image": rnd.randint(0, 20)}
        rr0 = dict(rr)
        res = rpol.route_image(req, insts, router, fan, rr)
        routes.append({"dims": [[i.width_px, i.height_px] for i in imgs], "pending": pend, "router": router.value,
                       "max_fanout": fan, "rr_in": rr0, "rr_out": rr,
                       "result": [[inst.id, list(idx)] for inst, idx in res]})

    batches = []
    stages = [rcore.StageKind.ENCODE, rcore.StageKind.PREPROCESS, rcore.StageKind.PREFILL]
    for case in range(200):
        items = []
        for s in range(rnd.randint(0, 20)):
            items.append(rengine.WorkItem(
                seq=s, request_id=rnd.randint(0, 5), stage=rnd.choice(stages), size_tokens=rnd.choice([1601, 3202, 4803, 6404, 576]),
                tiles=rnd.randint(1, 4), enqueue_ms=float(rnd.randint(0, 100)), ttft_slo_ms=float(rnd.choice([50, 100, 400])),
                deps=set([99]) if rnd.random() < 0.15 else set()))
        now = float(rnd.randint(0, 300))
        sched = rnd.choice(list(rpol.SchedulerKind))
        aging = rnd.choice([0.25, 0.5, 1.0])
        mb = {"encode": rnd.randint(1, 8), "preprocess": rnd.randint(1, 8), "prefill": rnd.randint(1, 4)}
        order = rpol.schedule_order(items, now, sched, aging)
        picked = rengine.form_batch(items, now, sched, aging, mb)
        batches.append({"items": [[it.seq, it.request_id, it.stage.value, it.size_tokens, it.tiles, it.enqueue_ms,
                                   it.ttft_slo_ms, sorted(it.deps)] for it in items],
                        "now": now, "scheduler": sched.value, "aging": aging, "max_batch": mb,
                        "order": order, "picked": picked})
    (OUT / "policies.json").write_text(json.dumps({"split": split_out, "route": routes, "batch": batches},
                                                  separators=(",", ":")))


def profile():
    """The reference's own calibrated profiles (profiles.py:400-470, default_profile :549) — the
    base (LLM-side fields) of the B200-measured profile exports, one per preset."""
    from lmmsim import profiles as rprof
    spec = rcore.get_model_spec("llama3.2-11b")
    prof = rprof.calibrate(rprof.load_calibration_targets(spec.name), spec)
    (OUT / "profile_llama.json").write_text(json.dumps(prof.to_dict(), indent=1))
    for name in ("internvl-26b", "llava-ov-7b", "llama3.2-90b", "llava-ov-72b", "nvlm-d-72b"):
        spec = rcore.get_model_spec(name)
        prof = rprof.default_profile(spec)
        (OUT / f"profile_{name}.json").write_text(json.dumps(prof.to_dict(), indent=1))


if __name__ == "__main__":
    profile()
    tiling()
    generator()
    policies()
    for p in sorted(OUT.glob("*.json")):
        print(p.name, p.stat().st_size)
