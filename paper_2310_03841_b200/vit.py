"""Checksum-protected Vision Transformers on the B200: `ProtectedLinear` and
ViT-B/16 / ViT-L/16 whose every Linear layer is a protected GEMM (K1).

The reference has no transformer (its stand-in is the toy GEMM pipeline,
/root/reference/pkg/src/gemmguard/model.py:191-235, with attention replaced by
token mixing, model.py:298-304).  The paper's object is a PyTorch wrapper
around the Linear layers of DeiT with attention left
unprotected; this module is that wrapper built B200-first:

* `ProtectedLinear(nn.Module)` holds the weight in torch layout [out, in], its
  offline checksum (K2: w_sum = sum over outputs, guard.offline_checksum,
  guard.py:142-160), the per-layer epsilon (mu, lo, hi; guard.EpsilonModel,
  guard.py:81-98) and calls K1 (`kernels.protected_gemm`): the GEMM, the
  per-row check d = X.w_sum + bias_sum - sum(Y) against the epsilon and an
  optional GELU fused into the epilogue AFTER the observed sum (the check
  covers the raw rounded output, guard.py:10-11).  Detection results stay on
  the device (`CheckResult`), so a forward never synchronises per layer.
* `ProtectedViT`: patch embedding as a protected GEMM over 16x16 patches,
  `depth` blocks of LN -> qkv -> SDPA attention -> proj -> residual + LN ->
  fc1 (+GELU) -> fc2 -> residual, final LN and a protected classifier head:
  4 * depth + 2 protected GEMMs (50 for ViT-B/16, 98 for ViT-L/16; the paper's
  DeiT-base also has 50 protected layers).  Residual updates and
  layer norms are one fused pass (`gg_add_layernorm`); attention runs through
  torch SDPA (unprotected).
* `resume`: the forward restarted at any protected layer from cached clean
  (residual, input) pairs — prefix reuse for injection campaigns (one trial
  per image, `campaign.py`).

Weights are random-initialised (no network for checkpoints); images are
synthetic.  Layer indices: 0 patch embed, 1 + 4b + {0 qkv, 1 proj, 2 fc1,
3 fc2} for block b, 4 * depth + 1 head.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch
import torch.nn.functional as F

from . import _lib as L
from . import kernels as K
from .calib import RunningStats

__all__ = ["ViTConfig", "VIT_B16", "VIT_L16", "ProtectedLinear", "ProtectedViT", "LAYER_ROLES"]

LAYER_ROLES = ("qkv", "proj", "fc1", "fc2")


@dataclass(frozen=True)
class ViTConfig:
    name: str = "vit_b16"
    image: int = 224
    patch: int = 16
    dim: int = 768
    depth: int = 12
    heads: int = 12
    mlp: int = 3072
    classes: int = 1000
    ln_eps: float = 1e-6

    @property
    def grid(self) -> int:
        return self.image // self.patch

    @property
    def tokens(self) -> int:
        return self.grid * self.grid + 1

    @property
    def patch_dim(self) -> int:
        return 3 * self.patch * self.patch

    @property
    def n_layers(self) -> int:
        return 4 * self.depth + 2

    def gemms(self, batch: int) -> list[tuple[str, int, int, int]]:
        """(name, M, N, K) of every protected GEMM of one forward at `batch` images."""
        m = batch * self.tokens
        g = [("patch_embed", batch * (self.tokens - 1), self.dim, self.patch_dim)]
        for b in range(self.depth):
            g += [(f"blk{b}.qkv", m, 3 * self.dim, self.dim), (f"blk{b}.proj", m, self.dim, self.dim),
                  (f"blk{b}.fc1", m, self.mlp, self.dim), (f"blk{b}.fc2", m, self.dim, self.mlp)]
        g.append(("head", batch, self.classes, self.dim))
        return g

    def flops_per_image(self) -> tuple[float, float]:
        """(protected-GEMM flops, attention flops) per image."""
        gemm = sum(2.0 * M * N * Kd for _, M, N, Kd in self.gemms(1))
        attn = self.depth * 2 * 2.0 * self.tokens * self.tokens * self.dim
        return gemm, attn


VIT_B16 = ViTConfig()
VIT_L16 = ViTConfig(name="vit_l16", dim=1024, depth=24, heads=16, mlp=4096)

class ProtectedLinear(torch.nn.Module):
    """y = x @ W.T + b as one protected GEMM launch (K1) with a device-resident check.

    `protected` False runs the unprotected instance of the same kernel family
    (the overhead baseline).  Until `set_epsilon` is called the float check
    flags nothing (thresholds +-inf); int8 layers use the exact rule d != 0.
    """

    def __init__(self, index: int, name: str, in_features: int, out_features: int, *, dtype: torch.dtype,
                 device, generator: torch.Generator | None = None, act: int = L.GG_ACT_NONE,
                 f32_mode: str = "3xtf32", init_scale: float = 1.0):
        super().__init__()
        self.index, self.name = index, name
        self.in_features, self.out_features = in_features, out_features
        self.act = act
        self.f32_mode = f32_mode
        self.protected = True
        w = torch.randn(out_features, in_features, device=device, generator=generator) * (
            init_scale / math.sqrt(in_features))
        if dtype == torch.int8:
            self.register_buffer("weight", torch.clamp(torch.round(w * 16.0), -127, 127).to(torch.int8))
            self.register_buffer("bias", torch.randint(-64, 65, (out_features,), device=device, generator=generator,
                                                       dtype=torch.int32))
        else:
            self.register_buffer("weight", w.to(dtype))
            self.register_buffer("bias", (0.02 * torch.randn(out_features, device=device, generator=generator)))
        self.mu, self.lo, self.hi = 0.0, -math.inf, math.inf
        self.result: K.CheckResult | None = None
        self.prepare()

    @property
    def integer(self) -> bool:
        return self.weight.dtype == torch.int8

    def prepare(self) -> None:
        """Offline checksum (K2, guard.offline_checksum) and its kernel encodings; weights are immutable."""
        prec = L.GG_P_I64 if self.integer else L.GG_P_F64
        self.w_sum, bsum = K.offline_checksum(self.weight, self.bias, prec)
        self.bias_sum = int(bsum.item()) if self.integer else float(bsum.item())
        self.aux = K.checksum_aux(self.w_sum, self.weight.dtype, self.f32_mode)
        self.w_split = (K.split_tf32x3(self.weight, 1)
                        if self.weight.dtype == torch.float32 and self.f32_mode == "3xtf32" else None)

    def set_epsilon(self, mu: float, lo: float, hi: float) -> None:
        self.mu, self.lo, self.hi = float(mu), float(lo), float(hi)

    def _kw(self, protect: bool) -> dict:
        kw = dict(protect=protect, f32_mode=self.f32_mode, w_split=self.w_split, act=self.act,
                  ws_key=("vit", self.name))
        if protect:
            kw.update(w_sum=self.w_sum, w_aux=self.aux, bias_sum=self.bias_sum, mu=self.mu,
                      lo=-1e300 if self.lo == -math.inf else self.lo, hi=1e300 if self.hi == math.inf else self.hi)
        return kw

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None, result: K.CheckResult | None = None,
                injections: torch.Tensor | None = None, protect: bool | None = None,
                pred_in: torch.Tensor | None = None, residual: torch.Tensor | None = None) -> torch.Tensor:
        """pred_in: x . w_sum computed by x's producer (kernels.add_layernorm with w_pred=self.aux).
        residual: the stored output is residual + y (the check covers y; no fused activation)."""
        p = self.protected if protect is None else protect
        kw = self._kw(p)
        if residual is not None:
            kw.pop("act")
        y, res = K.protected_gemm(x, self.weight, self.bias, out=out, result=result, injections=injections,
                                  pred_in=pred_in if p else None, residual=residual, **kw)
        self.result = res
        self.last_pred_in = pred_in if p else None
        self.last_residual = residual
        return y

    @property
    def pred_vector(self) -> torch.Tensor | None:
        """fp32 w_sum for a producer-side predicted sum (16-bit and single-pass tf32 kinds)."""
        if self.integer or (self.weight.dtype == torch.float32 and self.f32_mode == "3xtf32"):
            return None
        return self.aux

    def replay(self, x: torch.Tensor, y: torch.Tensor, rows: torch.Tensor, result: K.CheckResult,
               changed: torch.Tensor | None = None, granularity: str = "band") -> torch.Tensor:
        """K4 on this layer's last launch: recompute the bands of the flagged rows in place.

        granularity="tile": locate the faulty 256-column tiles of those bands by column
        checksums (kernels.locate_tiles) and recompute only them (kernels.replay_located);
        layers with a fused activation replay whole bands (their check needs the raw output)."""
        kw = self._kw(True)
        kw.pop("protect")
        residual = getattr(self, "last_residual", None)
        if residual is not None:
            kw.pop("act")
            kw["residual"] = residual
        if granularity == "tile" and self.act == L.GG_ACT_NONE and residual is None:
            ch, _ = K.replay_located(x, self.weight, self.bias, y, result, w_sum=self.w_sum,
                                     bias_sum=self.bias_sum, mu=kw["mu"], lo=kw["lo"], hi=kw["hi"],
                                     f32_mode=self.f32_mode, w_split=self.w_split, ws_key=kw["ws_key"],
                                     pred_in=getattr(self, "last_pred_in", None))
            if changed is not None:
                changed += ch
                return changed
            return ch
        if granularity not in ("band", "tile"):
            raise ValueError(f"unknown replay granularity {granularity!r}")
        return K.replay_tiles(x, self.weight, self.bias, y, rows, result, changed=changed,
                              pred_in=getattr(self, "last_pred_in", None), **kw)


def _located(lin: "ProtectedLinear", x: torch.Tensor, y: torch.Tensor, res: K.CheckResult) -> list:
    """The (128-row band, 256-column tile) pairs column checksums place the flagged faults in."""
    if lin.act != L.GG_ACT_NONE or getattr(lin, "last_residual", None) is not None:
        return []  # (the stored output is not the GEMM's alone)
    mask, _ = K.locate_tiles(x, lin.weight, lin.bias, y, res, mu=lin.mu)
    return [tuple(t) for t in mask.nonzero().tolist()]


@dataclass
class _Buffers:
    B: int
    patches: torch.Tensor
    e: torch.Tensor
    h: torch.Tensor
    a: torch.Tensor
    qkv: torch.Tensor
    o: torch.Tensor
    y: torch.Tensor
    f: torch.Tensor
    cls_in: torch.Tensor
    logits: torch.Tensor
    pred: torch.Tensor | None = None  # [B*T] predicted sums of the next GEMM, from the layer norm
    results: dict = field(default_factory=dict)
    o_view: torch.Tensor | None = None  # the proj input: the attention output itself when contiguous, else o
    h2: torch.Tensor | None = None  # the residual stream after proj when the GEMMs add it (fused_residual)


class ProtectedViT(torch.nn.Module):
    """ViT with every Linear layer protected (see the module docstring)."""

    def __init__(self, cfg: ViTConfig = VIT_B16, *, dtype: torch.dtype = torch.bfloat16, device="cuda",
                 seed: int = 0, f32_mode: str = "3xtf32"):
        super().__init__()
        self.cfg, self.dtype = cfg, dtype
        dev = torch.device(device)
        self.device_ = dev
        g = torch.Generator(device=dev).manual_seed(seed)
        D = cfg.dim
        fused_gelu = dtype in (torch.bfloat16, torch.float16)
        self.fused_gelu = fused_gelu
        # proj and fc2 store the residual stream's update h + y themselves (GG_ACT_RESIDUAL: the
        # check still covers y), so the layer norms after them read one matrix instead of two
        self.fused_residual = fused_gelu
        mk = lambda i, n, k_in, k_out, act=L.GG_ACT_NONE, s=1.0: ProtectedLinear(  # noqa: E731
            i, n, k_in, k_out, dtype=dtype, device=dev, generator=g, act=act, f32_mode=f32_mode, init_scale=s)
        layers = [mk(0, "patch_embed", cfg.patch_dim, D)]
        for b in range(cfg.depth):
            base = 1 + 4 * b
            layers += [mk(base, f"blk{b}.qkv", D, 3 * D), mk(base + 1, f"blk{b}.proj", D, D),
                       mk(base + 2, f"blk{b}.fc1", D, cfg.mlp, L.GG_ACT_GELU_TANH if fused_gelu else L.GG_ACT_NONE),
                       mk(base + 3, f"blk{b}.fc2", cfg.mlp, D)]
        layers.append(mk(cfg.n_layers - 1, "head", D, cfg.classes))
        self.linears = torch.nn.ModuleList(layers)
        self.register_buffer("cls", (0.02 * torch.randn(D, device=dev, generator=g)).to(dtype))
        self.register_buffer("pos", (0.02 * torch.randn(cfg.tokens, D, device=dev, generator=g)).to(dtype))
        # layer norms: depth x (ln1, ln2) + final; gamma / beta in fp32
        n_ln = 2 * cfg.depth + 1
        self.register_buffer("ln_g", 1.0 + 0.02 * torch.randn(n_ln, D, device=dev, generator=g))
        self.register_buffer("ln_b", 0.02 * torch.randn(n_ln, D, device=dev, generator=g))
        self._bufs: dict[int, _Buffers] = {}
        self.hooks = []  # callables (layer, result) after every protected launch (calibration)
        # Optionally the layer norms that feed qkv / fc1 also form those launches' predicted row
        # sums (pred_in), so K1's checksum warps hold no pipeline stage there.  Measured on ViT-B
        # b256: K1 qkv / fc1 -6 / -8 us per launch against the layer norm's extra work; with the
        # persistent layer norm (checksum vector in registers) still a wash (+0.8% / -0.9% in two
        # alternating runs, tools/pred_model_ab.py), so off by default.
        self.producer_pred = False

    # ------------------------------------------------------------- plumbing
    def layer(self, i: int) -> ProtectedLinear:
        return self.linears[i]

    def rows_per_image(self, i: int) -> int:
        if i == 0:
            return self.cfg.tokens - 1
        if i == self.cfg.n_layers - 1:
            return 1
        return self.cfg.tokens

    def buffers(self, B: int) -> _Buffers:
        bf = self._bufs.get(B)
        if bf is None:
            c, dev, dt = self.cfg, self.device_, self.dtype
            T, D = c.tokens, c.dim
            e = lambda *s: torch.empty(*s, device=dev, dtype=dt)  # noqa: E731
            bf = _Buffers(B=B, patches=e(B * (T - 1), c.patch_dim), e=e(B * (T - 1), D), h=e(B * T, D),
                          a=e(B * T, D), qkv=e(B * T, 3 * D), o=e(B * T, D), y=e(B * T, D), f=e(B * T, c.mlp),
                          cls_in=e(B, D), logits=torch.empty(B, c.classes, device=dev,
                                                             dtype=torch.int32 if dt == torch.int8 else dt),
                          pred=torch.empty(B * T, device=dev, dtype=torch.int64),
                          h2=e(B * T, D) if self.fused_residual else None)
            for lin in self.linears:
                M = B * self.rows_per_image(lin.index)
                bf.results[lin.index] = K.CheckResult.empty(M, lin.integer, dev)
            self._bufs[B] = bf
        return bf

    def set_protected(self, layers) -> None:
        """Protect only `layers` (selective protection, analysis.select_layers); the rest run unprotected."""
        chosen = set(layers)
        for lin in self.linears:
            lin.protected = lin.index in chosen

    def _feeds_pred(self, i: int, protect) -> bool:
        """Whether the layer norm writing layer i's input also forms its predicted sums."""
        lin = self.linears[i]
        on = lin.protected if protect is None else (protect and lin.protected)
        return bool(self.producer_pred and on and lin.pred_vector is not None)

    def _ln_into(self, i: int, protect, bf: _Buffers, h, y, g, b, h_out=None) -> None:
        """a = LN(h [+ y]) feeding protected layer i (with its pred_in when enabled)."""
        feeds = self._feeds_pred(i, protect)
        K.add_layernorm(h, y, g, b, self.cfg.ln_eps, ln_out=bf.a, h_out=h_out,
                        w_pred=self.linears[i].pred_vector if feeds else None, pred_out=bf.pred if feeds else None)
        bf.pred_valid = feeds

    def _lin(self, i: int, x: torch.Tensor, out: torch.Tensor, bf: _Buffers, protect: bool | None,
             injections: dict | None, pred: bool = False, residual: torch.Tensor | None = None) -> torch.Tensor:
        lin = self.linears[i]
        inj = injections.get(i) if injections else None
        use_pred = pred and getattr(bf, "pred_valid", False) and self._feeds_pred(i, protect)
        y = lin(x, out=out, result=bf.results[i], injections=inj,
                protect=None if protect is None else (protect and lin.protected),
                pred_in=bf.pred if use_pred else None, residual=residual)
        if lin.result is not None:
            for h in self.hooks:
                h(lin, lin.result)
        if i in getattr(self, "_replay_layers", ()):  # detect-then-replay (guard._replay semantics)
            self._maybe_replay(lin, x, y, bf)
        return y

    def _attention(self, bf: _Buffers) -> None:
        c = self.cfg
        B, T, H = bf.B, c.tokens, c.heads
        hd = c.dim // H
        qkv = bf.qkv.view(B, T, 3, H, hd)
        q, k, v = (qkv[:, :, j].transpose(1, 2) for j in range(3))
        o = F.scaled_dot_product_attention(q, k, v).transpose(1, 2)
        if o.is_contiguous():  # the attention kernel wrote [B, T, H, hd]: the proj input is a view
            bf.o_view = o.view(B * T, c.dim)
        else:
            bf.o.view(B, T, H, hd).copy_(o)
            bf.o_view = bf.o

    def _ln(self, j: int):
        return self.ln_g[j], self.ln_b[j]

    # -------------------------------------------------------------- forward
    def forward(self, images: torch.Tensor, *, protect: bool | None = None, injections: dict | None = None,
                cache: dict | None = None) -> torch.Tensor:
        """Logits [B, classes] of a batch of images [B, 3, H, W] (device).  Per-layer checks
        land in `buffers(B).results[i]`.  `cache` (a dict) receives the clean
        (residual, input) of every layer for `resume`."""
        B = images.shape[0]
        bf = self.buffers(B)
        c = self.cfg
        P, G = c.patch, c.grid
        if images.is_contiguous() and images.dtype == bf.patches.dtype and (P * images.element_size()) % 16 == 0:
            K.patchify(images, P, bf.patches)  # 16-byte copies (torch's permuted copy is element-wise)
        else:
            bf.patches.view(B, G, G, 3, P, P).copy_(images.view(B, 3, G, P, G, P).permute(0, 2, 4, 1, 3, 5))
        return self._run(bf, 0, protect, injections, cache)

    def resume(self, start: int, cache: dict, B: int, *, protect: bool | None = None,
               injections: dict | None = None) -> torch.Tensor:
        """The forward from protected layer `start` on, from a cache filled by `forward(cache=...)`."""
        return self._run(self.buffers(B), start, protect, injections, None, restore=cache)

    def _run(self, bf: _Buffers, start: int, protect, inj, cache, restore=None) -> torch.Tensor:
        c = self.cfg
        B, T, D = bf.B, c.tokens, c.dim
        eps = c.ln_eps
        h, a = bf.h, bf.a

        def save(i, resid, x):
            if cache is not None:
                pv = bf.pred.clone() if getattr(bf, "pred_valid", False) and x is a else None
                cache[i] = (None if resid is None else resid.clone(), x.clone(), pv)

        def load(i, resid, x):
            r, xi, pv = restore[i]
            if r is not None:
                resid.copy_(r)
            x.copy_(xi)
            bf.pred_valid = pv is not None
            if pv is not None:
                bf.pred.copy_(pv)

        if start == 0:
            save(0, None, bf.patches)
            self._lin(0, bf.patches, bf.e, bf, protect, inj)
            # position add, class token and the first layer norm in one pass (gg_embed_layernorm)
            feeds = self._feeds_pred(1, protect)
            K.embed_layernorm(bf.e, self.pos, self.cls, *self._ln(0), self.cfg.ln_eps, h_out=h, ln_out=bf.a,
                              w_pred=self.linears[1].pred_vector if feeds else None,
                              pred_out=bf.pred if feeds else None)
            bf.pred_valid = feeds
        for b in range(c.depth):
            base = 1 + 4 * b
            if start <= base:
                if start == base:
                    load(base, h, a)
                save(base, h, a)
                self._lin(base, a, bf.qkv, bf, protect, inj, pred=True)
                self._attention(bf)
            fr = self.fused_residual
            h2 = bf.h2 if fr else h  # the residual stream after proj
            if start <= base + 1:
                if start == base + 1:
                    load(base + 1, h, bf.o)
                    bf.o_view = bf.o
                save(base + 1, h, bf.o_view)
                if fr:  # h2 = h + proj(o) stored by the GEMM, then the layer norm of h2 alone
                    self._lin(base + 1, bf.o_view, h2, bf, protect, inj, residual=h)
                    self._ln_into(base + 2, protect, bf, h2, None, *self._ln(2 * b + 1))
                else:
                    self._lin(base + 1, bf.o_view, bf.y, bf, protect, inj)
                    self._ln_into(base + 2, protect, bf, h, bf.y, *self._ln(2 * b + 1), h_out=h)
            if start <= base + 2:
                if start == base + 2:
                    load(base + 2, h2, a)
                save(base + 2, h2, a)
                self._lin(base + 2, a, bf.f, bf, protect, inj, pred=True)
                if not self.fused_gelu:
                    bf.f.copy_(F.gelu(bf.f, approximate="tanh"))
            if start <= base + 3:
                if start == base + 3:
                    load(base + 3, h2, bf.f)
                save(base + 3, h2, bf.f)
                nxt = base + 4 if b + 1 < c.depth else None  # the next qkv (the final norm feeds the head's cls rows)
                if fr:  # h = h2 + fc2(f) stored by the GEMM
                    self._lin(base + 3, bf.f, h, bf, protect, inj, residual=h2)
                    y_add = None
                else:
                    self._lin(base + 3, bf.f, bf.y, bf, protect, inj)
                    y_add = bf.y
                if nxt is not None:
                    self._ln_into(nxt, protect, bf, h, y_add, *self._ln(2 * b + 2), h_out=h if y_add is not None else None)
                else:
                    K.add_layernorm(h, y_add, *self._ln(2 * b + 2), eps, ln_out=a, h_out=h if y_add is not None else None)
                    bf.pred_valid = False
        head = c.n_layers - 1
        if start == head:
            load(head, None, bf.cls_in)
        else:
            bf.cls_in.copy_(a.view(B, T, D)[:, 0])
        save(head, None, bf.cls_in)
        self._lin(head, bf.cls_in, bf.logits, bf, protect, inj)
        return bf.logits

    # ------------------------------------------------------ detect + replay
    def enable_replay(self, layers=None, max_replays: int = 3, granularity: str = "band") -> None:
        """Detect-then-replay (guard._replay, guard.py:575-604) on `layers` (default: all):
        after a protected launch whose check triggered, K4 recomputes only the
        128-row bands holding flagged rows with the clean weight (granularity="tile":
        only the 256-column tiles of those bands that column checksums place the
        fault in); the host reads one device scalar per protected layer (the
        reference checks per layer too)."""
        self._replay_layers = set(range(self.cfg.n_layers)) if layers is None else set(layers)
        self._max_replays = max_replays
        self._replay_granularity = granularity
        self.replay_events = []

    def disable_replay(self) -> None:
        self._replay_layers = set()

    def _maybe_replay(self, lin: ProtectedLinear, x, y, bf: _Buffers) -> None:
        res = lin.result
        if res is None or not bool(res.triggered.item()):
            return
        from .errors import GuardError

        for attempt in range(1, self._max_replays + 1):
            changed = lin.replay(x, y, res.flags.clone(), res,
                                 granularity=getattr(self, "_replay_granularity", "band"))
            n_changed = int(changed.item())
            if n_changed == 0:  # the recompute reproduced the flagged bytes: numerical, accepted
                self.replay_events.append((lin.index, "replay_numerical", attempt))
                return
            if not bool(res.triggered.item()):
                self.replay_events.append((lin.index, "replay", attempt))
                return
        raise GuardError(f"layer {lin.index}: replay budget ({self._max_replays}) exhausted; "
                         f"persistent fault suspected in (band, column tile) {_located(lin, x, y, res)}")

    # ---------------------------------------------------------- calibration
    @torch.no_grad()
    def calibrate(self, batches, confidence: float) -> dict[int, tuple[float, float, float]]:
        """Per-layer epsilon from clean batches (guard.calibrate_epsilon, guard.py:277-356):
        the fused check's d of every row folds into device-resident running
        moments (gg_running_stats); thresholds mu -/+ z sigma."""
        stats = {lin.index: RunningStats(self.device_) for lin in self.linears if not lin.integer}
        saved = [(lin.mu, lin.lo, lin.hi) for lin in self.linears]
        for lin in self.linears:
            lin.set_epsilon(0.0, -math.inf, math.inf)

        def hook(lin, res):
            if lin.index in stats:
                stats[lin.index].update(res.d)

        self.hooks.append(hook)
        try:
            for images in batches:
                self.forward(images, protect=True)
        finally:
            self.hooks.remove(hook)
        out = {}
        for lin, old in zip(self.linears, saved):
            if lin.index in stats:
                mu, lo, hi = stats[lin.index].epsilon(confidence)
                lin.set_epsilon(mu, lo, hi)
                out[lin.index] = (mu, lo, hi)
            else:
                lin.set_epsilon(0.0, 0.0, 0.0)
        return out

    def role_groups(self) -> dict[str, list[int]]:
        """Layer indices by role: patch_embed, qkv, proj, fc1, fc2, head."""
        d = self.cfg.depth
        groups = {"patch_embed": [0]}
        for j, role in enumerate(LAYER_ROLES):
            groups[role] = [1 + 4 * b + j for b in range(d)]
        groups["head"] = [self.cfg.n_layers - 1]
        return groups

    def flagged_rows(self, B: int) -> torch.Tensor:
        """Device int64 [n_layers]: flagged rows of the last forward's checks per layer."""
        bf = self.buffers(B)
        return torch.cat([bf.results[i].nflag.long() for i in range(self.cfg.n_layers)])
