"""Host-side stage API and oracle vs golden vectors produced by the REFERENCE itself
(tests/golden/make_golden.py ran lmmsim in the authoring container).  Bit-exact."""

import json
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import tiling as otiling
from paper_2502_00937_b200 import batcher, core, policies, workload

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def tiling_gold():
    return json.loads((GOLD / "tiling.json").read_text())


def _spec_from_gold(name, entry):
    T, tok, cap, thumb = entry["spec"]
    return core.ModelSpec(name=name, architecture=core.Architecture.DEC_ONLY, tile_edge_px=T, tokens_per_tile=tok,
                          max_tiles_per_image=cap, thumbnail_tile=bool(thumb))


def test_tiling_product_matches_reference(tiling_gold):
    n = 0
    for name, entry in tiling_gold.items():
        spec = _spec_from_gold(name, entry)
        for w, h, tiles, toks in entry["rows"]:
            if tiles < 0:
                with pytest.raises(core.SpecError):
                    core.tile_count(w, h, spec)
                with pytest.raises(core.SpecError):
                    core.ImageSpec.from_dims(w, h, spec)
                continue
            assert core.tile_count(w, h, spec) == tiles
            assert core.image_tokens(w, h, spec) == toks
            n += 1
    assert n > 30000


def test_tiling_oracle_c_matches_reference(tiling_gold):
    for name, entry in tiling_gold.items():
        T, tok, cap, thumb = entry["spec"]
        rows = np.array(entry["rows"], dtype=np.int64)
        ok = (rows[:, 0] <= 2**31 - 1)
        rows = rows[ok]
        plan = otiling.tile_plan(rows[:, 0], rows[:, 1], T, tok, cap, bool(thumb), 0)
        expect = np.where(rows[:, 2] < 0, 0, rows[:, 2])
        np.testing.assert_array_equal(plan["tiles"], expect)
        assert plan["bad"] == int((rows[:, 2] < 0).sum())
        np.testing.assert_array_equal(np.diff(plan["tile_off"]), expect)
        np.testing.assert_array_equal(plan["tok_off"], plan["tile_off"] * tok)
        # python literal restatement too
        for w, h, tiles, _ in entry["rows"][:400]:
            assert otiling.tile_count_py(w, h, T, cap, bool(thumb)) == tiles


def test_generator_matches_reference():
    cases = json.loads((GOLD / "generator.json").read_text())
    for case in cases:
        spec = core.get_model_spec(case["model"])
        kw = dict(case["kw"])
        if "images_per_request" in kw:
            kw["images_per_request"] = {int(k): v for k, v in kw["images_per_request"].items()}
        bursts = tuple(workload.BurstEpisode(*b) for b in case["burst"])
        cfg = workload.GeneratorConfig(model=spec, seed=case["seed"], burst_episodes=bursts, **kw)
        reqs = workload.generate(cfg, case["horizon_ms"])
        assert len(reqs) == len(case["requests"])
        for r, g in zip(reqs, case["requests"]):
            assert r.arrival_ms == g[0] and r.text_tokens == g[1] and r.output_tokens == g[2]
            assert r.service_id == g[3]
            assert [[i.width_px, i.height_px, i.tiles, i.image_tokens] for i in r.images] == g[4]
            assert r.total_image_tokens == g[5] and r.total_tiles == g[6]


@pytest.fixture(scope="module")
def pol_gold():
    return json.loads((GOLD / "policies.json").read_text())


def test_split_by_tiles_matches_reference(pol_gold):
    for tiles, n, expect in pol_gold["split"]:
        assert policies.split_by_tiles(tiles, n) == expect


def test_route_image_matches_reference(pol_gold):
    spec = core.get_model_spec("llama3.2-11b")
    for case in pol_gold["route"]:
        imgs = tuple(core.ImageSpec.from_dims(w, h, spec) for w, h in case["dims"])
        req = core.Request(id=0, arrival_ms=0.0, text_tokens=10, images=imgs, output_tokens=1)
        insts = [SimpleNamespace(id=k, pending_image_tokens=p, pending_text_tokens=0)
                 for k, p in enumerate(case["pending"])]
        rr = dict(case["rr_in"])
        res = policies.route_image(req, insts, policies.RouterKind(case["router"]), case["max_fanout"], rr)
        assert [[inst.id, list(idx)] for inst, idx in res] == case["result"]
        assert rr == case["rr_out"]


def test_form_batch_matches_reference(pol_gold):
    for case in pol_gold["batch"]:
        items = [batcher.WorkItem(seq=s, request_id=r, stage=core.StageKind(st), size_tokens=sz, tiles=t,
                                  enqueue_ms=e, ttft_slo_ms=slo, deps=set(deps))
                 for s, r, st, sz, t, e, slo, deps in case["items"]]
        sched = policies.SchedulerKind(case["scheduler"])
        assert policies.schedule_order(items, case["now"], sched, case["aging"]) == case["order"]
        assert batcher.form_batch(items, case["now"], sched, case["aging"], case["max_batch"]) == case["picked"]
