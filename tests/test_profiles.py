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
    assert ref["encode_ms_per_tile"] == {"1": pytest.approx(700.0 / 64)}
    assert ref["prefill_self_ms_per_token"] == base["prefill_self_ms_per_token"]
    # the reference's own loader (authoring container only) prices stages with the measured constants
    if not Path("/root/reference/pkg/src").exists():
        pytest.skip("reference not mounted")
    sys.path.insert(0, "/root/reference/pkg/src")
    from lmmsim import core as rcore
    from lmmsim import profiles as rprofiles
    rp = rprofiles.LatencyProfile.from_dict(ref, rcore.get_model_spec("llama3.2-11b"))
    assert rp.encode_latency(64, 1) == pytest.approx(700.0)
    assert rp.preprocess_latency(100, base["ref_cpu_cores"]) == pytest.approx(1.0)
