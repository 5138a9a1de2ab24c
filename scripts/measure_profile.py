#!/usr/bin/env python
"""Measure the B200 latency profile of the image path and export it.

    python scripts/measure_profile.py [--model llama3.2-11b] [--scale profiles/scale_*.json ...]

Writes profiles/measured_<model>.json (MeasuredProfile) and profiles/measured_<model>.reference.json
(the reference's profile schema, profiles.py:268-326, LLM-side fields from
tests/golden/profile_<model>.json, image-stage fields measured), which the reference's own
LatencyProfile.from_dict loads (tests/test_profiles.py).  ``--scale`` takes bench.py JSON lines
at N GPUs to fill dp_efficiency (throughput / (N x one-GPU throughput)).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3.2-11b")
    ap.add_argument("--scale", nargs="*", default=[])
    ap.add_argument("--export-only", action="store_true",
                    help="no measurement: re-export the committed profiles/measured_<model>.json (CPU)")
    ap.add_argument("--from-model", default=None,
                    help="with --export-only: take the measurement of a preset with the same image path "
                         "(encoder block and tiling), e.g. llama3.2-11b for llama3.2-90b")
    args = ap.parse_args()
    from paper_2502_00937_b200 import core
    from paper_2502_00937_b200.profiles import MeasuredProfile
    spec = core.get_model_spec(args.model)
    if args.export_only:
        src = core.get_model_spec(args.from_model or args.model)
        same = (src.encoder == spec.encoder and src.tile_edge_px == spec.tile_edge_px
                and src.max_tiles_per_image == spec.max_tiles_per_image and src.thumbnail_tile == spec.thumbnail_tile)
        if not same:
            raise SystemExit(f"{src.name} and {spec.name} do not share the image path")
        d = json.loads(open(os.path.join(ROOT, "profiles", f"measured_{src.name}.json")).read())
        if src.name != spec.name:
            d["model"] = spec.name
            d.setdefault("meta", {})["measured_as"] = src.name
        prof = MeasuredProfile.from_dict(d, spec)
    else:
        import torch  # noqa: F401
        from paper_2502_00937_b200.executor import ImagePathExecutor
        from paper_2502_00937_b200.profiles import measure_profile
        prof = measure_profile(ImagePathExecutor(spec, seed=0))
    lines = [json.loads(open(p).read().strip().splitlines()[-1]) for p in args.scale]
    one = [d["value"] for d in lines if d.get("n_gpus") == 1]
    if one:
        for d in lines:
            if d.get("n_gpus", 1) > 1:
                prof.dp_efficiency[int(d["n_gpus"])] = round(d["value"] / (d["n_gpus"] * one[0]), 4)
    out = os.path.join(ROOT, "profiles", f"measured_{spec.name}.json")
    prof.save(out)
    # LLM-side fields from the reference's own calibrated profile of the preset (tests/golden,
    # made by running the reference: make_golden.py)
    gold = os.path.join(ROOT, "tests", "golden", f"profile_{spec.name}.json")
    if not os.path.exists(gold):
        gold = os.path.join(ROOT, "tests", "golden", "profile_llama.json")
    base = json.loads(open(gold).read())
    if base.get("model") == spec.name:
        ref = prof.to_reference_profile(base)
        open(os.path.join(ROOT, "profiles", f"measured_{spec.name}.reference.json"), "w").write(
            json.dumps(ref, indent=2) + "\n")
    print(json.dumps({"model": spec.name, **prof.to_dict()}))


if __name__ == "__main__":
    main()
