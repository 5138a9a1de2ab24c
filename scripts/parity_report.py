"""Parity report: the CUDA path against the fp32 CPU oracle at full model depth, per image
(relative L2 error of the packed embeddings; tolerance 1e-2), plus the bit-exact checks of K0 / K1.
Prints one JSON object (profiles/r02/r02_parity.json).  InternViT-6B's weights are drawn on the GPU
(5.5 B parameters), so its fp32 oracle runs with torch on the GPU (TF32 off)."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import encoders as oenc, preprocess as oprep, tiling as otiling
from paper_2502_00937_b200 import core, ops
from paper_2502_00937_b200.encoders import k_pad_of
from paper_2502_00937_b200.executor import ImagePathExecutor, stage_images

torch.set_num_threads(len(os.sched_getaffinity(0)))
report = {"tolerance": 1e-2, "metric": "per-image ||y - y_oracle|| / ||y_oracle|| over the packed embeddings",
          "weights": "random init (seeded), Mllama gates randomised", "configs": {}}
cases = {"llama3.2-11b": [(560, 560), (1000, 500), (1400, 900), (1120, 1120)],
         "llava-clip-l14-336": [(336, 336), (800, 600), (300, 1000)],
         "vit-b16-224": [(224, 224)] * 4,
         "llava-ov-7b": [(384, 384), (1000, 700), (700, 1400)],
         "internvl-26b": [(448, 448), (900, 800), (1300, 500)]}
for name, dims in cases.items():
    spec = core.get_model_spec(name)
    enc = spec.encoder
    rng = np.random.default_rng(7)
    imgs = [rng.integers(0, 256, (h, w, 3), dtype=np.uint8) for w, h in dims]
    ex = ImagePathExecutor(spec, seed=3)
    out = ex.encode(stage_images(imgs))
    torch.cuda.synchronize()
    plan = otiling.tile_plan([d[0] for d in dims], [d[1] for d in dims], spec.tile_edge_px, spec.tokens_per_tile,
                             spec.max_tiles_per_image, spec.thumbnail_tile, enc.resize_mode)
    scale, shift = oprep.norm_constants(enc.mean, enc.std)
    ref_bits = oprep.preprocess(imgs, plan, spec.tile_edge_px, enc.patch_px, k_pad_of(spec), enc.resize_mode,
                                spec.thumbnail_tile, scale, shift)
    # K1 on the device, bit for bit
    b = stage_images(imgs)
    dplan = ops.tile_plan(b.w, b.h, spec)
    dev_bits = ops.preprocess(b.src, b.src_off, b.w, b.h, dplan["tile_off"], dplan["geom"], len(dims),
                              int(plan["tile_off"][-1]), spec, k_pad_of(spec), torch.from_numpy(scale).cuda(),
                              torch.from_numpy(shift).cuda()).view(torch.int16).cpu().numpy().view(np.uint16)
    t0 = time.time()
    wdev = ex.weights["patch_w"].device
    ref = oenc.encode(torch.from_numpy(oprep.bf16_bits_to_f32(ref_bits)).to(wdev), plan, ex.weights, spec).cpu()
    got = out.embeds.float().cpu()
    offs = plan["tok_off"]
    rel = []
    for i in range(len(dims)):
        a, e = int(offs[i]), int(offs[i + 1])
        rel.append(float((got[a:e] - ref[a:e]).norm() / ref[a:e].norm()))
    report["configs"][name] = {
        "images": [list(d) for d in dims], "tiles": [int(x) for x in plan["tiles"]],
        "tok_offsets_equal": out.tok_offsets.cpu().tolist() == plan["tok_off"].tolist(),
        "preprocess_bf16_mismatches": int((dev_bits != ref_bits).sum()), "preprocess_values": int(ref_bits.size),
        "rel_err_per_image": [round(r, 6) for r in rel], "max_rel_err": round(max(rel), 6),
        "oracle_s": round(time.time() - t0, 1), "oracle_device": str(wdev),
        "layers": enc.layers + getattr(enc, "global_layers", 0)}
    print(name, report["configs"][name], file=sys.stderr, flush=True)
print(json.dumps(report))
