"""Checksum-protected Swin-B (BASELINE.json configs[4]): int8 MLP layers and
bf16 attention / merge / embed / head layers, every Linear a protected GEMM (K1).

Architecture (Swin-B, 224^2): 4x4 patch embedding (48 -> 128, layer norm),
stages of depths (2, 2, 18, 2) with (4, 8, 16, 32) heads at 56^2 / 28^2 /
14^2 / 7^2 tokens and widths 128 / 256 / 512 / 1024, 7x7 window attention
with a learned relative position bias, every second block on windows shifted
by 3 (with the cross-window mask), patch merging (2x2 concat, layer norm,
4C -> 2C without bias) between stages, final layer norm, average pool and the
1000-class head: 1 + 4 * 24 + 3 + 1 = 101 protected GEMMs.

Mixed precision (the split named in configs[4]): the MLP GEMMs fc1 / fc2 run
on int8 tensor cores (kind::i8, int32 accumulation) with per-tensor symmetric
scales — their check is the reference's exact int64 rule (d != 0,
guard.py:192-194), so every corrupted output is detected — and the other
GEMMs run in bf16 with a calibrated per-layer epsilon.  Quantise / dequantise
/ GELU around the int8 layers, window partition, shifts and attention (torch
SDPA with the bias and mask as an additive attention mask) are unprotected
glue (only the Linear layers carry checksums).

Random-initialised weights (there is no network for checkpoints), synthetic
images.  `forward` supports detect-then-replay through `ProtectedViT`'s
mechanism (K4 on the flagged bands of the layer whose check fired).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn.functional as F

from . import kernels as K
from .calib import RunningStats
from .vit import ProtectedLinear

__all__ = ["SwinConfig", "SWIN_B", "ProtectedSwin"]


@dataclass(frozen=True)
class SwinConfig:
    name: str = "swin_b"
    image: int = 224
    patch: int = 4
    embed: int = 128
    depths: tuple = (2, 2, 18, 2)
    heads: tuple = (4, 8, 16, 32)
    window: int = 7
    mlp_ratio: int = 4
    classes: int = 1000
    ln_eps: float = 1e-5

    def stage_dims(self):
        """(resolution, width) per stage."""
        r, c = self.image // self.patch, self.embed
        out = []
        for _ in self.depths:
            out.append((r, c))
            r, c = r // 2, c * 2
        return out

    def gemms(self, batch: int) -> list[tuple[str, int, int, int, str]]:
        """(name, M, N, K, precision) of every protected GEMM of one forward."""
        g = [("patch_embed", batch * (self.image // self.patch) ** 2, self.embed, 3 * self.patch ** 2, "bf16")]
        for s, ((r, c), d) in enumerate(zip(self.stage_dims(), self.depths)):
            m = batch * r * r
            for b in range(d):
                g += [(f"s{s}.b{b}.qkv", m, 3 * c, c, "bf16"), (f"s{s}.b{b}.proj", m, c, c, "bf16"),
                      (f"s{s}.b{b}.fc1", m, self.mlp_ratio * c, c, "int8"),
                      (f"s{s}.b{b}.fc2", m, c, self.mlp_ratio * c, "int8")]
            if s < len(self.depths) - 1:
                g.append((f"s{s}.merge", batch * (r // 2) ** 2, 2 * c, 4 * c, "bf16"))
        g.append(("head", batch, self.classes, self.stage_dims()[-1][1], "bf16"))
        return g


SWIN_B = SwinConfig()


def _relative_index(w: int) -> torch.Tensor:
    coords = torch.stack(torch.meshgrid(torch.arange(w), torch.arange(w), indexing="ij")).flatten(1)  # [2, w*w]
    rel = coords[:, :, None] - coords[:, None, :] + (w - 1)
    return rel[0] * (2 * w - 1) + rel[1]  # [w*w, w*w]


def _shift_mask(r: int, w: int, s: int, device) -> torch.Tensor:
    """[nW, w*w, w*w] additive mask (0 / -inf) of the shifted-window partition."""
    img = torch.zeros(r, r, device=device)
    cnt = 0
    for hs in (slice(0, -w), slice(-w, -s), slice(-s, None)):
        for ws in (slice(0, -w), slice(-w, -s), slice(-s, None)):
            img[hs, ws] = cnt
            cnt += 1
    win = img.view(r // w, w, r // w, w).permute(0, 2, 1, 3).reshape(-1, w * w)
    diff = win[:, None, :] - win[:, :, None]
    return torch.where(diff != 0, float("-inf"), 0.0)


class _Int8Linear:
    """Per-tensor symmetric quantisation around an int8 ProtectedLinear: y = (q(x) q(W)^T + q(b)) s_x s_w."""

    def __init__(self, lin: ProtectedLinear, w_fp: torch.Tensor, b_fp: torch.Tensor):
        self.lin = lin
        self.s_w = float(w_fp.abs().max()) / 127.0
        lin.weight.copy_(torch.clamp(torch.round(w_fp / self.s_w), -127, 127).to(torch.int8))
        self.b_fp = b_fp
        self.s_x = None

    def set_input_scale(self, s_x: float):
        self.s_x = float(s_x)
        self.lin.bias.copy_(torch.round(self.b_fp / (self.s_x * self.s_w)).to(torch.int32))
        self.lin.prepare()  # checksum of the quantised weight / bias

    def quantize(self, x: torch.Tensor) -> torch.Tensor:
        return torch.clamp(torch.round(x.float() / self.s_x), -127, 127).to(torch.int8)

    def dequantize(self, y: torch.Tensor) -> torch.Tensor:
        return y.float() * (self.s_x * self.s_w)


class ProtectedSwin(torch.nn.Module):
    """Swin-B with every Linear protected (module docstring)."""

    def __init__(self, cfg: SwinConfig = SWIN_B, *, device="cuda", seed: int = 0, int8_mlp: bool = True):
        super().__init__()
        self.cfg = cfg
        dev = torch.device(device)
        self.device_ = dev
        g = torch.Generator(device=dev).manual_seed(seed)
        self.int8_mlp = int8_mlp
        layers, self.quant = [], {}
        idx = 0

        def lin(name, k_in, k_out, dtype=torch.bfloat16, bias=True):
            nonlocal idx
            pl = ProtectedLinear(idx, name, k_in, k_out, dtype=dtype, device=dev, generator=g)
            if not bias:
                pl.bias.zero_()
                pl.prepare()
            layers.append(pl)
            idx += 1
            return pl

        def mlp_lin(name, k_in, k_out):
            if not int8_mlp:
                return lin(name, k_in, k_out)
            w = torch.randn(k_out, k_in, device=dev, generator=g) / math.sqrt(k_in)
            b = 0.02 * torch.randn(k_out, device=dev, generator=g)
            pl = lin(name, k_in, k_out, dtype=torch.int8)
            self.quant[pl.index] = _Int8Linear(pl, w, b)
            return pl

        self.embed = lin("patch_embed", 3 * cfg.patch ** 2, cfg.embed)
        self.blocks, self.merges = [], []
        ln_count = 1  # patch norm
        for s, ((r, c), d) in enumerate(zip(cfg.stage_dims(), cfg.depths)):
            stage = []
            for b in range(d):
                stage.append(dict(
                    qkv=lin(f"s{s}.b{b}.qkv", c, 3 * c), proj=lin(f"s{s}.b{b}.proj", c, c),
                    fc1=mlp_lin(f"s{s}.b{b}.fc1", c, cfg.mlp_ratio * c), fc2=mlp_lin(f"s{s}.b{b}.fc2", cfg.mlp_ratio * c, c),
                    ln1=ln_count, ln2=ln_count + 1, shift=(b % 2 == 1) and r > cfg.window, heads=cfg.heads[s],
                    bias=0.02 * torch.randn((2 * cfg.window - 1) ** 2, cfg.heads[s], device=dev, generator=g)))
                ln_count += 2
            self.blocks.append(stage)
            if s < len(cfg.depths) - 1:
                self.merges.append(dict(lin=lin(f"s{s}.merge", 4 * c, 2 * c, bias=False), ln=ln_count, dim=4 * c))
                ln_count += 1
        self.head = lin("head", cfg.stage_dims()[-1][1], cfg.classes)
        self.final_ln = ln_count
        ln_count += 1
        self.linears = torch.nn.ModuleList(layers)
        maxd = 4 * cfg.stage_dims()[-1][1]
        self.ln_g = 1.0 + 0.02 * torch.randn(ln_count, maxd, device=dev, generator=g)
        self.ln_b = 0.02 * torch.randn(ln_count, maxd, device=dev, generator=g)
        self.rel_index = _relative_index(cfg.window).to(dev)
        self._masks = {}
        self.hooks = []
        self.results = {}
        self._last_keys = []
        self._replay_layers = set()

    @property
    def n_layers(self) -> int:
        return len(self.linears)

    # ------------------------------------------------------------- glue
    def _ln(self, x: torch.Tensor, j: int, dim: int) -> torch.Tensor:
        return F.layer_norm(x.float(), (dim,), self.ln_g[j, :dim], self.ln_b[j, :dim], self.cfg.ln_eps).to(
            torch.bfloat16)

    def _run(self, lin: ProtectedLinear, x: torch.Tensor, protect: bool, injections: dict | None) -> torch.Tensor:
        inj = injections.get(lin.index) if injections else None
        M = x.shape[0]
        key = (lin.index, M)
        self._last_keys.append(key)
        res = self.results.get(key)
        if res is None and protect:
            res = K.CheckResult.empty(M, lin.integer, self.device_)
            self.results[key] = res
        y = lin(x, result=res, injections=inj, protect=protect and lin.protected)
        if lin.result is not None:
            for h in self.hooks:
                h(lin, lin.result)
            if lin.index in self._replay_layers:
                self._maybe_replay(lin, x, y)
        return y

    def _linear(self, lin: ProtectedLinear, x: torch.Tensor, protect: bool, injections) -> torch.Tensor:
        """bf16 in, bf16 (or fp32 dequantised) out; int8 layers quantise around the GEMM."""
        q = self.quant.get(lin.index)
        if q is None:
            return self._run(lin, x, protect, injections)
        if q.s_x is None:  # first use: the input scale from this (clean) activation
            q.set_input_scale(float(x.float().abs().max()) / 127.0)
        return q.dequantize(self._run(lin, q.quantize(x), protect, injections))

    def _mask(self, r: int, shift: int):
        key = (r, shift)
        if key not in self._masks:
            self._masks[key] = _shift_mask(r, self.cfg.window, shift, self.device_)
        return self._masks[key]

    def _attention(self, qkv: torch.Tensor, B: int, r: int, c: int, heads: int, shift: bool, bias_tab) -> torch.Tensor:
        w = self.cfg.window
        s = w // 2 if shift else 0
        x = qkv.view(B, r, r, 3 * c)
        if s:
            x = torch.roll(x, shifts=(-s, -s), dims=(1, 2))
        nw = r // w
        x = x.view(B, nw, w, nw, w, 3, heads, c // heads).permute(5, 0, 1, 3, 6, 2, 4, 7)
        x = x.reshape(3, B * nw * nw, heads, w * w, c // heads)
        bias = bias_tab[self.rel_index.view(-1)].view(w * w, w * w, heads).permute(2, 0, 1)  # [h, n, n]
        mask = bias.unsqueeze(0).to(torch.bfloat16)
        if s:
            m = self._mask(r, s)  # [nW, n, n]
            mask = (bias.unsqueeze(0) + m.unsqueeze(1)).repeat(B, 1, 1, 1).to(torch.bfloat16)
        o = F.scaled_dot_product_attention(x[0], x[1], x[2], attn_mask=mask)  # [B nW, h, n, hd]
        o = o.view(B, nw, nw, heads, w, w, c // heads).permute(0, 1, 4, 2, 5, 3, 6).reshape(B, r, r, c)
        if s:
            o = torch.roll(o, shifts=(s, s), dims=(1, 2))
        return o.reshape(B * r * r, c).contiguous()

    # ---------------------------------------------------------- forward
    @torch.no_grad()
    def forward(self, images: torch.Tensor, *, protect: bool = True, injections: dict | None = None) -> torch.Tensor:
        c0 = self.cfg
        B = images.shape[0]
        self._last_keys = []
        P, r0 = c0.patch, c0.image // c0.patch
        x = images.to(torch.bfloat16).view(B, 3, r0, P, r0, P).permute(0, 2, 4, 1, 3, 5).reshape(B * r0 * r0, -1)
        h = self._ln(self._linear(self.embed, x.contiguous(), protect, injections), 0, c0.embed)
        for s, ((r, c), stage) in enumerate(zip(c0.stage_dims(), self.blocks)):
            for blk in stage:
                a = self._ln(h, blk["ln1"], c)
                qkv = self._linear(blk["qkv"], a, protect, injections)
                o = self._attention(qkv, B, r, c, blk["heads"], blk["shift"], blk["bias"])
                h = (h.float() + self._linear(blk["proj"], o, protect, injections).float()).to(torch.bfloat16)
                a = self._ln(h, blk["ln2"], c)
                f = F.gelu(self._linear(blk["fc1"], a, protect, injections).float(), approximate="tanh")
                h = (h.float() + self._linear(blk["fc2"], f.to(torch.bfloat16), protect, injections).float()).to(
                    torch.bfloat16)
            if s < len(self.merges):
                mg = self.merges[s]
                v = h.view(B, r, r, c)
                cat = torch.cat([v[:, 0::2, 0::2], v[:, 1::2, 0::2], v[:, 0::2, 1::2], v[:, 1::2, 1::2]], dim=-1)
                cat = self._ln(cat.reshape(-1, 4 * c), mg["ln"], 4 * c)
                h = self._linear(mg["lin"], cat, protect, injections)
        r, c = c0.stage_dims()[-1]
        hf = self._ln(h, self.final_ln, c).view(B, r * r, c).float().mean(dim=1).to(torch.bfloat16)
        return self._linear(self.head, hf.contiguous(), protect, injections)

    # --------------------------------------------------- calibration / replay
    @torch.no_grad()
    def calibrate(self, batches, confidence: float) -> None:
        """Per-layer epsilon of the bf16 layers from clean batches (device running moments);
        the int8 layers fix their activation scales on the first batch and use the exact rule."""
        stats = {lin.index: RunningStats(self.device_) for lin in self.linears if not lin.integer}
        for lin in self.linears:
            if not lin.integer:
                lin.set_epsilon(0.0, -math.inf, math.inf)

        def hook(lin, res):
            if lin.index in stats:
                stats[lin.index].update(res.d)

        self.hooks.append(hook)
        try:
            for b in batches:
                self.forward(b, protect=True)
        finally:
            self.hooks.remove(hook)
        for lin in self.linears:
            if lin.index in stats:
                lin.set_epsilon(*stats[lin.index].epsilon(confidence))

    def enable_replay(self, layers=None, max_replays: int = 3, granularity: str = "band") -> None:
        """Detect-then-replay on `layers` (default: all); granularity as ProtectedViT.enable_replay."""
        self._replay_layers = set(range(self.n_layers)) if layers is None else set(layers)
        self._max_replays = max_replays
        self._replay_granularity = granularity
        self.replay_events = []

    def disable_replay(self) -> None:
        self._replay_layers = set()

    def _maybe_replay(self, lin: ProtectedLinear, x, y) -> None:
        res = lin.result
        if not bool(res.triggered.item()):
            return
        from .errors import GuardError

        for attempt in range(1, self._max_replays + 1):
            n = int(lin.replay(x, y, res.flags.clone(), res,
                               granularity=getattr(self, "_replay_granularity", "band")).item())
            if n == 0:
                self.replay_events.append((lin.index, "replay_numerical", attempt))
                return
            if not bool(res.triggered.item()):
                self.replay_events.append((lin.index, "replay", attempt))
                return
        raise GuardError(f"layer {lin.index}: replay budget ({self._max_replays}) exhausted")

    def flagged_rows(self) -> dict[int, int]:
        """Flagged rows per protected layer of the last forward (only layers that flagged)."""
        out = {}
        for key in self._last_keys:
            res = self.results.get(key)
            if res is not None and int(res.nflag.item()):
                out[key[0]] = int(res.nflag.item())
        return out
