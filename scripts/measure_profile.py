#!/usr/bin/env python
"""Measure the B200 latency profile of the image path and export it.

    python scripts/measure_profile.py [--model llama3.2-11b] [--scale profiles/scale_*.json ...]

Writes profiles/measured_<model>.json (MeasuredProfile) and profiles/measured_<model>.reference.json
(the reference's profile schema, profiles.py:268-326, LLM-side fields from
tests/golden/profile_llama.json, image-stage fields measured), which the reference's own
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
    args = ap.parse_args()
    import torch
    from paper_2502_00937_b200 import core
    from paper_2502_00937_b200.executor import ImagePathExecutor
    from paper_2502_00937_b200.profiles import measure_profile
    spec = core.get_model_spec(args.model)
    prof = measure_profile(ImagePathExecutor(spec, seed=0))
    lines = [json.loads(open(p).read().strip().splitlines()[-1]) for p in args.scale]
    one = [d["value"] for d in lines if d.get("n_gpus") == 1]
    if one:
        for d in lines:
            if d.get("n_gpus", 1) > 1:
                prof.dp_efficiency[int(d["n_gpus"])] = round(d["value"] / (d["n_gpus"] * one[0]), 4)
    out = os.path.join(ROOT, "profiles", f"measured_{spec.name}.json")
    prof.save(out)
    base = json.loads(open(os.path.join(ROOT, "tests", "golden", "profile_llama.json")).read())
    if base.get("model") == spec.name:
        ref = prof.to_reference_profile(base)
        open(os.path.join(ROOT, "profiles", f"measured_{spec.name}.reference.json"), "w").write(
            json.dumps(ref, indent=2) + "\n")
    print(json.dumps({"model": spec.name, "device": torch.cuda.get_device_name(), **prof.to_dict()}))


if __name__ == "__main__":
    main()
