"""pytest plugin: the reference's ``lmmsim`` package with its image-path symbols replaced by
the product's, so the reference's OWN unit tests run against this repo's drop-in modules.

Used only by tests/test_reference_suite.py (CPU, authoring container: it needs the
read-only reference tree at /root/reference, which the GPU box does not have).

* ``lmmsim.core``      IS ``paper_2502_00937_b200.core`` (reference core.py:13-189)
* ``lmmsim.workload``  reference module; generator and trace I/O swapped for the product's
                       (workload.py:28-121, :124-296); ``summarize`` / ``fit_tail_exponent``
                       stay the reference's (out of scope)
* ``lmmsim.policies``  reference module; ``split_by_tiles`` / ``route_image`` /
                       ``schedule_order`` / ``schedule_next`` swapped (policies.py:91-179);
                       autoscaler / placement stay the reference's (out of scope)
* ``lmmsim.engine``    reference event loop (out of scope) driving the product's
                       ``WorkItem`` / ``encode_shard`` / ``form_batch`` (engine.py:73-114)

Swaps happen before the next module imports, so the reference's ``from .x import y``
bindings pick up the product symbols too: the simulator itself runs on the product code.
"""

from __future__ import annotations

import importlib
import importlib.util
import os
import sys

REF_PKG = os.environ.get("LMMSIM_REF", "/root/reference/pkg/src/lmmsim")
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2502_00937_b200 import batcher, core, policies, workload  # noqa: E402

SWAPS = {
    "workload": (workload, ["TraceError", "TRACE_COLUMNS", "TraceRecord", "TraceLoadResult", "load_trace",
                            "write_trace", "BurstEpisode", "GeneratorConfig", "DEFAULT_IMAGES_PER_REQUEST",
                            "sample_power_law", "generate", ("_parse_dims", "parse_dims")]),
    "policies": (policies, ["split_by_tiles", "route_image", "schedule_order", "schedule_next"]),
    "engine": (batcher, ["WorkItem", "encode_shard", "form_batch"]),
}
SWAPPED: dict[str, list[str]] = {}


def _install() -> None:
    spec = importlib.util.spec_from_file_location("lmmsim", os.path.join(REF_PKG, "__init__.py"),
                                                  submodule_search_locations=[REF_PKG])
    pkg = importlib.util.module_from_spec(spec)
    sys.modules["lmmsim"] = pkg
    spec.loader.exec_module(pkg)
    sys.modules["lmmsim.core"] = core
    pkg.core = core
    for name in ("workload", "profiles", "policies", "engine"):
        mod = importlib.import_module(f"lmmsim.{name}")
        src, names = SWAPS.get(name, (None, []))
        for entry in names:
            dst_name, src_name = entry if isinstance(entry, tuple) else (entry, entry)
            setattr(mod, dst_name, getattr(src, src_name))
            SWAPPED.setdefault(name, []).append(dst_name)


_install()


def pytest_report_header(config):
    return ["lmmsim shim: core -> paper_2502_00937_b200.core; "
            + "; ".join(f"{m}: {', '.join(v)}" for m, v in SWAPPED.items())]


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(pytest_report_header(None)[0])
