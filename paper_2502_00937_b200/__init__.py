"""B200-native image path of a ModServe-style multimodal server (arXiv 2502.00937).

Host-side stage API (pure Python, importable without a GPU) mirrors the reference `lmmsim`:
``core`` (specs, tiling counts, requests), ``policies`` (image routing, batch ordering),
``batcher`` (WorkItem, form_batch), ``workload`` (synthetic images / traces), ``profiles``
(measured-latency profile).  The compute path (``ops``, ``encoders``, ``executor``, ``dp``)
runs hand-written sm_100a kernels from libmmk.so through a C ABI (include/mmk.h); importing
it without the built library raises ImportError — there is no CPU fallback.
"""

__version__ = "0.1.0"

from .core import (  # noqa: F401
    Architecture, EncoderSpec, ImageSpec, ModelSpec, Request, SLOSpec, SpecError, StageKind,
    get_model_spec, image_tokens, load_model_specs, request_totals, tile_count,
)
