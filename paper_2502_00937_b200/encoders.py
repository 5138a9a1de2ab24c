"""Vision encoders of the image path, executed as libmmk kernels on one B200.

Replaces the modelled encode stage (reference LatencyProfile.encode_latency,
pkg/src/lmmsim/profiles.py:136-145, called from engine.py:693-703) with the real forward:

  patches -> K2 patch GEMM -> embedding assembly + LN_pre -> L x [ K3 LN -> K4 QKV GEMM ->
  K5 varlen attention -> K6 O-proj GEMM + (gated) residual -> K3 LN -> K7 FC1 GEMM + GELU ->
  K8 FC2 GEMM + (gated) residual (+ intermediate capture) ] -> K9 pack

Families (EncoderSpec.family):
* "clip"   pre-LN ViT (ViT-B/16-224, CLIP ViT-L/14-336 as used by LLaVA: layer -2, no CLS;
           SigLIP-400M of LLaVA-OneVision; InternViT-6B of InternVL / NVLM: RMSNorm, QK-norm,
           layer scale folded into the O-proj / FC2 weights, pixel-shuffled output)
* "mllama" Llama-3.2-Vision encoder: gated tile embeddings, 32 local + 8 gated global layers,
           output = [final | interleaved hidden_states[3,7,15,23,30]] (7680 wide;
           EncoderSpec.out_layers_of fixes which hidden state index i names)

Residual stream in fp32 (HBM), GEMM operands in bf16, fp32 accumulation in TMEM.
Weights are random-initialised from a seed (no checkpoints in this environment).
"""

from __future__ import annotations

import math
import os

import torch

from . import ops
from .core import ModelSpec, SpecError

from .weights import K_ALIGN, init_weights, k_pad_of  # noqa: F401  (re-exported)


# Narrow encoders (ViT-B, d 768: its reference-default batch 8 is a launch-latency-bound 1 ms
# step) keep the LN kernels: the fold saves HBM traffic such steps do not spend (measured -2 %).
# The choice is per encoder, never per batch, so an image's embedding does not depend on which
# batch it was encoded in (replay.py --verify re-encodes shards alone and compares bit for bit).
FOLD_MIN_HIDDEN = 1024


class DeviceEncoder:
    """Device-resident weights + the forward of one encoder over a ragged batch of tiles."""

    def __init__(self, spec: ModelSpec, weights: dict, device="cuda", fold_ln: bool | None = None):
        enc = spec.encoder
        if enc is None:
            raise SpecError(f"{spec.name}: no encoder block")
        if enc.head_dim > 128:
            from ._lib import ProfileError
            raise ProfileError(f"{spec.name}: head_dim {enc.head_dim} not supported by the attention kernel")
        self.spec, self.enc, self.device = spec, enc, torch.device(device)
        # head_dim below a kernel size (SigLIP 72) runs as zero-padded heads of the next size (80):
        # zero Q/K columns leave the scores unchanged (scale stays head_dim^-0.5), zero V columns
        # give zero output columns, which meet zero columns of the O-projection
        self.hd = enc.head_dim
        self.hd_pad = 64 if enc.head_dim <= 64 else 80 if enc.head_dim <= 80 else 128
        # FFN widths that are not a multiple of 256 (SigLIP 4304) pad with zero units (act(0) = 0)
        self.ffn_pad = -(-enc.ffn // 256) * 256 if enc.ffn % 256 else enc.ffn
        # LayerNorm folded into the GEMMs (mmk_gemm_bf16_ln): every LN whose input comes from a
        # residual GEMM; MMK_LN_FOLD=0 / =1 forces the separate LayerNorm kernel / the fold (A/B runs)
        if fold_ln is None:
            env = os.environ.get("MMK_LN_FOLD")
            fold_ln = enc.hidden >= FOLD_MIN_HIDDEN if env is None else env != "0"
        self.fold_ln = bool(fold_ln) and enc.hidden % 32 == 0
        self.P = (spec.tile_edge_px // enc.patch_px) ** 2
        self.S = self.P + int(enc.cls_token)  # encoder tokens per tile
        self.k_pad = k_pad_of(spec)
        dev = self.device
        bf = lambda t: t.to(dev, torch.bfloat16).contiguous()  # noqa: E731
        f32 = lambda t: None if t is None else t.to(dev, torch.float32).contiguous()  # noqa: E731
        d = enc.hidden
        pw = torch.zeros(d, self.k_pad)
        pw[:, :weights["patch_w"].shape[1]] = weights["patch_w"]
        self.patch_w = bf(pw)
        self.patch_b = f32(weights.get("patch_b"))
        self.cls, self.pos = f32(weights.get("cls")), f32(weights["pos"])
        self.pre_ln = (f32(weights["pre_ln_w"]), f32(weights["pre_ln_b"])) if enc.pre_ln else (None, None)
        self.post_ln = (f32(weights["post_ln_w"]), f32(weights.get("post_ln_b")))
        self.rms = enc.norm == "rms"
        if enc.qk_norm and enc.head_dim not in (64, 80, 128):
            raise SpecError(f"{spec.name}: QK-norm with padded heads (head_dim {enc.head_dim}) is not supported")

        def folded(w, g, b, bias):
            """(W * gamma in bf16, c1 = row sums of it, c2 = beta W^T + bias): a LayerNorm with
            (gamma, beta) in front of the GEMM W folded into the GEMM (see mmk_gemm_bf16_ln); an
            RMSNorm (beta None) has mean 0 in the epilogue, so c1 is unused and c2 = bias."""
            wf = (w.double() * g.double()[None, :]).to(torch.bfloat16)
            c1 = wf.double().sum(1)
            c2 = torch.zeros(w.shape[0], dtype=torch.float64, device=w.device)
            if b is not None:
                c2 = c2 + w.double() @ b.double()
            if bias is not None:
                c2 = c2 + bias.double()
            return bf(wf), f32(c1.float()), f32(c2.float())

        def scaled(w, b, ls):
            """Layer scale lambda (per output channel) folded into the branch's last GEMM."""
            if ls is None:
                return w, b
            return ls[:, None] * w, (ls * b if b is not None else None)

        H, hd, hdp, ff, ffp = enc.heads, self.hd, self.hd_pad, enc.ffn, self.ffn_pad

        def pad_heads_rows(w):  # [3*H*hd, ...] -> [3*H*hdp, ...] (zero rows per head)
            if w is None or hd == hdp:
                return w
            v = w.reshape(3, H, hd, *w.shape[1:])
            out = torch.zeros(3, H, hdp, *w.shape[1:], dtype=w.dtype)
            out[:, :, :hd] = v
            return out.reshape(3 * H * hdp, *w.shape[1:])

        def pad_heads_cols(w):  # [d, H*hd] -> [d, H*hdp]
            if hd == hdp:
                return w
            out = torch.zeros(w.shape[0], H, hdp, dtype=w.dtype)
            out[:, :, :hd] = w.reshape(w.shape[0], H, hd)
            return out.reshape(w.shape[0], H * hdp)

        def pad_ffn_rows(w):  # [ff, ...] -> [ffp, ...]
            if w is None or ff == ffp:
                return w
            out = torch.zeros(ffp, *w.shape[1:], dtype=w.dtype)
            out[:ff] = w
            return out

        def pad_ffn_cols(w):  # [d, ff] -> [d, ffp]
            if ff == ffp:
                return w
            out = torch.zeros(w.shape[0], ffp, dtype=w.dtype)
            out[:, :ff] = w
            return out

        def block(pre, gated):
            qkv_w, qkv_b = pad_heads_rows(weights[pre + "qkv_w"]), pad_heads_rows(weights.get(pre + "qkv_b"))
            fc1_w, fc1_b = pad_ffn_rows(weights[pre + "fc1_w"]), pad_ffn_rows(weights[pre + "fc1_b"])
            o_w, o_b = scaled(pad_heads_cols(weights[pre + "o_w"]), weights.get(pre + "o_b"), weights.get(pre + "ls1"))
            fc2_w, fc2_b = scaled(pad_ffn_cols(weights[pre + "fc2_w"]), weights[pre + "fc2_b"], weights.get(pre + "ls2"))
            L = {
                "ln1": (f32(weights[pre + "ln1_w"]), f32(weights.get(pre + "ln1_b"))),
                "qkv_w": bf(qkv_w), "qkv_b": f32(qkv_b),
                "o_w": bf(o_w), "o_b": f32(o_b),
                "ln2": (f32(weights[pre + "ln2_w"]), f32(weights.get(pre + "ln2_b"))),
                "fc1_w": bf(fc1_w), "fc1_b": f32(fc1_b),
                "fc2_w": bf(fc2_w), "fc2_b": f32(fc2_b),
                "gate_attn": math.tanh(float(weights[pre + "gate_attn"])) if gated else 1.0,
                "gate_ffn": math.tanh(float(weights[pre + "gate_ffn"])) if gated else 1.0,
                "qk_norm": (f32(weights[pre + "q_norm"]), f32(weights[pre + "k_norm"])) if enc.qk_norm else None,
            }
            if self.fold_ln:
                L["qkv_f"] = folded(qkv_w, weights[pre + "ln1_w"], weights.get(pre + "ln1_b"), qkv_b)
                L["fc1_f"] = folded(fc1_w, weights[pre + "ln2_w"], weights.get(pre + "ln2_b"), fc1_b)
            return L

        self.layers = [block(f"l{i}.", False) for i in range(enc.layers)]
        self.global_layers = [block(f"g{i}.", True) for i in range(enc.global_layers)]
        if enc.family == "mllama":
            tpos = math.tanh(float(weights["pos_gate"]))
            self.pos_scale, self.tile_pos_scale = 1.0 - tpos, tpos
            self.pre_scale = math.tanh(float(weights["pre_gate"]))
            self.tile_pos = f32(weights["tile_pos"])
            self.pre_tile = f32(weights["pre_tile"])
            # post-tile embedding folded with its gate: added inside the LN_post kernel
            self.post_tile_scaled = f32(weights["post_tile"] * math.tanh(float(weights["post_gate"])))
            self.slots = weights["tile_pos"].shape[1]
        mean = torch.tensor(enc.mean, dtype=torch.float64)
        std = torch.tensor(enc.std, dtype=torch.float64)
        self.norm_scale = (1.0 / (255.0 * std)).to(torch.float32).to(dev)
        self.norm_shift = (-mean / std).to(torch.float32).to(dev)

    # ------------------------------------------------------------------ layers
    def _block(self, L, resid, x_buf, qkv_buf, h_buf, cu, n_seq, max_s, aux=None, sum_sq=0.0, ln=None, xr=None,
               stats_next=False, a_buf=None):
        """One pre-LN block.  Folded LayerNorms (self.fold_ln): ``ln`` = (stats, mr) buffers; LN1
        is folded when ``xr`` (the bf16 copy of the residual the previous FC2 wrote) is given, LN2
        always; with ``stats_next`` the FC2 also emits the next block's LN statistics.  Returns the
        bf16 copy of the updated residual (for the next block's folded LN1) or None."""
        enc = self.enc
        T, d = resid.shape
        if xr is not None:  # LN1 folded: QKV = act-free epilogue rstd * (acc - mu c1) + c2
            wf, c1, c2 = L["qkv_f"]
            ops.gemm(xr, wf, ops.EPI_BF16, bias=c2, out=qkv_buf, ln_mr=ln[1], ln_c1=c1)
        else:
            ops.layernorm(resid, *L["ln1"], enc.norm_eps, out=x_buf)
            ops.gemm(x_buf, L["qkv_w"], ops.EPI_BF16, bias=L["qkv_b"], out=qkv_buf)
        if L["qk_norm"] is not None:
            ops.qk_rmsnorm(qkv_buf, enc.heads * self.hd_pad, *L["qk_norm"], enc.norm_eps)
        a_buf = x_buf if a_buf is None else a_buf  # attention output (H * padded head_dim columns)
        ops.attention(qkv_buf, cu, n_seq, max_s, enc.heads, self.hd_pad, out=a_buf, scale=self.hd ** -0.5,
                      sum_sq_seqlen=sum_sq * self.hd / self.hd_pad)
        if ln is not None:
            # the O-proj writes the residual's bf16 copy into the (now free) Q columns of qkv_buf
            # and its LN statistics; FC1 consumes the copy with LN2 folded in
            xr2 = qkv_buf[:, :d]
            ops.gemm(a_buf, L["o_w"], ops.EPI_RESID_F32, bias=L["o_b"], out=resid, gate=L["gate_attn"], aux=xr2,
                     ln_stats_out=ln[0])
            ops.ln_stats_finalize(ln[0], T, d, enc.norm_eps, out=ln[1], rms=self.rms)
            wf, c1, c2 = L["fc1_f"]
            ops.gemm(xr2, wf, ops.ACT_EPI[enc.act], bias=c2, out=h_buf, ln_mr=ln[1], ln_c1=c1)
        else:
            ops.gemm(a_buf, L["o_w"], ops.EPI_RESID_F32, bias=L["o_b"], out=resid, gate=L["gate_attn"])
            ops.layernorm(resid, *L["ln2"], enc.norm_eps, out=x_buf)
            ops.gemm(x_buf, L["fc1_w"], ops.ACT_EPI[enc.act], bias=L["fc1_b"], out=h_buf)
        if ln is not None and stats_next:
            # the bf16 copy goes to the capture buffer when this layer is captured, else to x_buf
            # (free: the attention output was consumed by the O-proj)
            dst = aux if aux is not None else x_buf
            ops.gemm(h_buf, L["fc2_w"], ops.EPI_RESID_F32, bias=L["fc2_b"], out=resid, gate=L["gate_ffn"], aux=dst,
                     ln_stats_out=ln[0])
            ops.ln_stats_finalize(ln[0], T, d, enc.norm_eps, out=ln[1], rms=self.rms)
            return dst
        ops.gemm(h_buf, L["fc2_w"], ops.EPI_RESID_F32, bias=L["fc2_b"], out=resid, gate=L["gate_ffn"], aux=aux)
        return None

    def _run_layers(self, layers, resid, x_buf, qkv_buf, h_buf, cu, n_seq, max_s, sum_sq, aux_of=lambda i: None):
        """A stack of blocks; with fold_ln only the stack's first LN1 runs as a LayerNorm kernel."""
        T, d = resid.shape
        a_buf = None
        if self.enc.heads * self.hd_pad != d:  # padded heads: the attention output is wider than d
            a_buf = torch.empty(T, self.enc.heads * self.hd_pad, dtype=torch.bfloat16, device=resid.device)
        ln = None
        if self.fold_ln:
            ln = (torch.empty(T, d // 32, 2, dtype=torch.float32, device=resid.device),
                  torch.empty(T, 2, dtype=torch.float32, device=resid.device))
        xr = None
        for i, L in enumerate(layers):
            xr = self._block(L, resid, x_buf, qkv_buf, h_buf, cu, n_seq, max_s, aux=aux_of(i), sum_sq=sum_sq, ln=ln,
                             xr=xr, stats_next=i + 1 < len(layers), a_buf=a_buf)

    def forward(self, patches: torch.Tensor, total_tiles: int, cu_seqlens: torch.Tensor, n_seq: int, max_seqlen: int,
                tile_image=None, tile_slot=None, image_ar=None, out_alloc=None, sum_sq_seqlen: float = 0.0) -> torch.Tensor:
        """patches [total_tiles*P, k_pad] bf16 -> packed embeddings for the LLM prefill.
        cu_seqlens int32 [n_seq+1] token offsets of the attention sequences (one per image).
        out_alloc(rows, width) -> bf16 tensor: destination of the packed output, possibly in the
        LLM-backend GPU's memory (peer view); the pack then streams whole rows over NVLink."""
        enc, P, d, S = self.enc, self.P, self.enc.hidden, self.S
        dev = patches.device
        T = total_tiles * S
        patch_out = ops.gemm(patches, self.patch_w, ops.EPI_F32, bias=self.patch_b)
        if enc.family == "mllama":
            resid = ops.embed_tokens(patch_out, total_tiles, P, self.cls, self.pos, self.pos_scale, *self.pre_ln,
                                     enc.norm_eps, tile_image=tile_image, tile_slot=tile_slot, image_ar=image_ar,
                                     tile_pos=self.tile_pos, tile_pos_scale=self.tile_pos_scale,
                                     pre_tile=self.pre_tile, pre_scale=self.pre_scale, slots=self.slots)
        else:
            resid = ops.embed_tokens(patch_out, total_tiles, P, self.cls, self.pos, 1.0, *self.pre_ln, enc.norm_eps)
        del patch_out
        x_buf = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
        qkv_buf = torch.empty(T, 3 * enc.heads * self.hd_pad, dtype=torch.bfloat16, device=dev)
        h_buf = torch.empty(T, self.ffn_pad, dtype=torch.bfloat16, device=dev)
        if enc.family == "clip":
            n_run = enc.layers if enc.out_layer == -1 else enc.layers + 1 + enc.out_layer
            self._run_layers(self.layers[:n_run], resid, x_buf, qkv_buf, h_buf, cu_seqlens, n_seq, max_seqlen,
                             sum_sq_seqlen)
            # emitted = hidden_states[out_layer] as transformers' CLIPVisionModel numbers them
            # (modeling_clip.py: post_layernorm touches only the pooled CLS, never the sequence)
            drop = 1 if enc.drop_cls else 0
            if enc.pixel_shuffle:  # InternVL: CLS dropped, 2x2 patch groups -> 4 d channels
                side = self.spec.tile_edge_px // enc.patch_px
                dst = out_alloc(total_tiles * (side // 2) ** 2, 4 * d) if out_alloc is not None else None
                return ops.pack_pixel_shuffle(resid, total_tiles, side, S, drop, out=dst)
            dst = out_alloc(total_tiles * (S - drop), d) if out_alloc is not None else None
            return ops.pack_drop_cls(resid, total_tiles, S, drop, out=dst)
        # ---------------- mllama
        # intermediate capture: the FC2 epilogue of the layer whose output is the requested hidden
        # state writes a bf16 copy (EncoderSpec.out_layers_of: Meta "input of layer i" or
        # transformers-5 "output of layer i")
        outs = list(enc.out_layers)
        inter = torch.empty(len(outs), T, d, dtype=torch.bfloat16, device=dev)

        def aux_of(i):
            k = enc.capture_after(i)
            return inter[k] if k is not None else None
        self._run_layers(self.layers, resid, x_buf, qkv_buf, h_buf, cu_seqlens, n_seq, max_seqlen, sum_sq_seqlen,
                         aux_of=aux_of)
        # layernorm_post + gated post-tile positional embedding, in place on the fp32 stream
        ops.layernorm(resid, *self.post_ln, enc.norm_eps, out=resid, out_f32=True, tile_add=self.post_tile_scaled,
                      tile_image=tile_image, image_table=image_ar, tile_slot=tile_slot, rows_per_tile=P + 1,
                      slots=self.slots)
        self._run_layers(self.global_layers, resid, x_buf, qkv_buf, h_buf, cu_seqlens, n_seq, max_seqlen,
                         sum_sq_seqlen)
        del x_buf, qkv_buf, h_buf
        if out_alloc is not None:
            return ops.pack_mllama(resid, inter, out=out_alloc(T, d * (1 + len(outs))), peer=True)
        return ops.pack_mllama(resid, inter)
