"""MeasuredProfile keeps the reference LatencyProfile seam (profiles.py:128-145) and exports into
the reference profile schema (profiles.py:268-326)."""

import json
import sys
from pathlib import Path

import pytest

from paper_2502_00937_b200 import core
from paper_2502_00937_b200.profiles import MeasuredProfile, ProfileError

GOLD = Path(__file__).resolve().parent / "golden"
LLAMA = core.get_model_spec("llama3.2-11b")


def _prof():
    return MeasuredProfile(model=LLAMA, encode_points=[(2, 30.0), (8, 100.0), (64, 700.0)],
                           preprocess_ms_per_tile=0.01, preprocess_floor_ms=0.0)


def test_encode_latency_semantics():
    p = _prof()
    assert p.encode_latency(8, 1) == pytest.approx(100.0)
    assert p.encode_latency(5, 1) == pytest.approx(65.0)       # interpolated
    assert p.encode_latency(72, 1) == pytest.approx(700 + 8 * 600 / 56)  # extrapolated
    assert p.encode_latency(1, 1) == pytest.approx(30 - 35.0 / 3)
    with pytest.raises(ProfileError):
        p.encode_latency(0, 1)
    with pytest.raises(ProfileError):
        p.encode_latency(4, 2)   # not measured
    with pytest.raises(ProfileError):
        p.encode_latency(4, 3)   # not supported by the spec


def test_preprocess_latency_semantics():
    p = _prof()
    assert p.preprocess_latency(0, 4) == 0.0
    assert p.preprocess_latency(10, 4) == pytest.approx(0.1)
    with pytest.raises(ProfileError):
        p.preprocess_latency(1, 0)


def test_roundtrip_and_reference_export(tmp_path):
    p = _prof()
    p.save(tmp_path / "m.json")
    q = MeasuredProfile.from_dict(json.loads((tmp_path / "m.json").read_text()), LLAMA)
    assert q.encode_points == p.encode_points
    with pytest.raises(ProfileError):
        MeasuredProfile.from_dict(p.to_dict(), core.get_model_spec("internvl-26b"))
    base = json.loads((GOLD / "profile_llama.json").read_text())
    ref = p.to_reference_profile(base)
    # every TP degree of the spec: TP-1 measured, TP > 1 as its data-parallel equivalent
    assert ref["encode_ms_per_tile"] == {"1": pytest.approx(700.0 / 64), "2": pytest.approx(350.0 / 64),
                                         "4": pytest.approx(175.0 / 64), "8": pytest.approx(87.5 / 64)}
    assert ref["prefill_self_ms_per_token"] == base["prefill_self_ms_per_token"]
    # the reference's own loader (authoring container only) prices stages with the measured constants
    if not Path("/root/reference/pkg/src").exists():
        pytest.skip("reference not mounted")
    sys.path.insert(0, "/root/reference/pkg/src")
    from lmmsim import core as rcore
    from lmmsim import profiles as rprofiles
    rp = rprofiles.LatencyProfile.from_dict(ref, rcore.get_model_spec("llama3.2-11b"))
    assert rp.encode_latency(64, 1) == pytest.approx(700.0)
    assert rp.encode_latency(64, 4) == pytest.approx(175.0)  # select_sharding picking TP-4 no longer fails
    assert rp.preprocess_latency(100, base["ref_cpu_cores"]) == pytest.approx(1.0)


def test_batch_priced_from_its_tile_histogram():
    """encode_latency_images: per-image cost of each tile count (super-linear in tiles), DP over
    GPUs with the measured efficiency; unknown tile counts scale quadratically in tokens."""
    p = MeasuredProfile(model=LLAMA, encode_points=[(8, 100.0)], preprocess_ms_per_tile=0.01,
                        tile_costs={1: 3.0, 2: 8.0, 4: 20.0}, dp_efficiency={2: 0.9})
    assert p.encode_latency_images([1, 1, 2, 4]) == pytest.approx(34.0)
    assert p.encode_latency_images([3]) == pytest.approx(8.0 * (3 / 2) ** 2)  # nearest measured: 2 (tie -> lower)
    assert p.encode_latency_images([4, 4], tp=2) == pytest.approx(40.0 / 1.8)
    with pytest.raises(ProfileError):
        p.encode_latency_images([1], tp=4)
    with pytest.raises(ProfileError):
        p.encode_latency_images([])
    q = MeasuredProfile.from_dict(json.loads(json.dumps(p.to_dict())), LLAMA)
    assert q.tile_costs == p.tile_costs and q.dp_efficiency == p.dp_efficiency


PROFILES = Path(__file__).resolve().parent.parent / "profiles"


@pytest.mark.parametrize("model", ["llama3.2-11b", "llama3.2-90b", "internvl-26b", "nvlm-d-72b", "llava-ov-7b",
                                   "llava-ov-72b"])
def test_committed_b200_profile_loads_in_the_reference(model):
    """The B200-measured profile (scripts/measure_profile.py on a B200) in the reference schema,
    loaded by the reference's own LatencyProfile.from_dict (profiles.py:299-326); LLM-side fields
    from the reference's calibrated profile of the same preset (tests/golden/profile_<model>.json)."""
    measured = PROFILES / f"measured_{model}.reference.json"
    if not measured.exists():
        pytest.skip("no B200-measured profile committed")
    spec = core.get_model_spec(model)
    ref = json.loads(measured.read_text())
    assert ref["model"] == model
    mp = MeasuredProfile.from_dict(json.loads((PROFILES / f"measured_{model}.json").read_text()), spec)
    assert len(mp.encode_points) >= 3 and len(mp.tile_costs) >= 3
    if model.startswith("llama3.2"):
        assert mp.tile_costs[4] > 2 * mp.tile_costs[2] > 0  # super-linear in tiles (cross-tile attention)
    if not Path("/root/reference/pkg/src").exists():
        pytest.skip("reference not mounted")
    sys.path.insert(0, "/root/reference/pkg/src")
    from lmmsim import core as rcore
    from lmmsim import profiles as rprofiles
    rp = rprofiles.LatencyProfile.from_dict(ref, rcore.get_model_spec(model))
    t, ms = mp.encode_points[-1]
    assert rp.encode_latency(t, 1) == pytest.approx(ms, rel=1e-6)
    for tp in (2, 4, 8):
        assert rp.encode_latency(t, tp) < rp.encode_latency(t, 1)
