"""Batched, device-resident injection campaigns on a protected model.

The reference runs one host-driven inference per injection: `injected_forward`
re-runs the whole model from layer 0 on a scratch copy (injector.py:224-287),
`run_campaign` stratifies n trials per layer with a per-trial RNG seeded by
(seed, layer, k) (injector.py:451-565) and `evaluate_detection` counts a
trial as a true positive when the output changed class AND the injected
layer's check fired (guard.py:700-792).  On the B200 the same trial semantics
run as a batch:

* one trial per image of a batch: every image carries its own single output
  fault in its own rows of the injected layer's launch (faults in distinct
  rows never interact: the check is per row, guard.py:188-215, and images are
  independent in a ViT), applied in the GEMM epilogue before the observed
  sums (K1's in-epilogue injection; the reference corrupts the stored output
  before the check, guard.py:515-523);
* prefix reuse: the clean forward caches every protected layer's (residual,
  input), and a trial batch restarts at its layer (`ProtectedViT.resume`);
* mismatch (argmax change against the clean prediction, injector.py:318) and
  detection (any flagged row of the image at the injected layer) are
  computed on the device and folded into int64 counters per layer, which K5
  all-reduces across ranks (`distributed.reduce_counters`); nothing but the
  counters and compact per-trial records leaves the device;
* sampling follows `sample_injection`'s rules for the output location
  (injector.py:131-210): per trial an RNG from SeedSequence((seed, layer, k)),
  per attempt element -> mode -> bit, rejecting no-op flips and corrupted
  values outside the layer's profiled clean range [lo, hi], at most 64
  attempts (a trial with none is skipped, as SamplingError skips it in
  guard.py:705-709).  Attempts are drawn on the host in rounds of four per
  trial and validated on the device against the clean outputs.  The trial's
  image is fixed by k (k mod the golden-set size) instead of a drawn sample
  id, so that a batch holds one trial per image.

Work units are (layer, trial block); `plan_units` balances them over ranks
by suffix cost (a trial at an early layer recomputes more of the model).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from . import distributed as Dd
from . import kernels as K
from .calib import RunningRange

__all__ = ["ViTCampaign", "CampaignTally", "wilson_interval", "plan_units", "select_golden_images", "FIELDS",
           "BF16_FIELDS"]

FIELDS = ("injections", "mismatches", "true_positives", "false_negatives", "benign_detections", "true_negatives",
          "skipped", "loss_delta_fx")
# loss shifts are summed as int64 fixed point (2^-32 units) so that K5's all-reduce stays an
# order-independent integer sum; a non-finite or huge shift counts as +/-LOSS_CLAMP
LOSS_FX = 2.0**32
LOSS_CLAMP = 1.0e6
# (mantissa, exponent) bits per device dtype; bfloat16 is an extension (the reference has no bf16 tag)
BF16_FIELDS = {torch.bfloat16: (7, 8), torch.float16: (10, 5), torch.float32: (23, 8)}
MAX_RETRIES = 64  # injector.py:53
ROUND = 4


def wilson_interval(k: int, n: int, z: float = 1.959963984540054) -> tuple[float, float]:
    """Wilson score interval of a binomial proportion k / n (95% by default)."""
    if n == 0:
        return (0.0, 1.0)
    p = k / n
    d = 1.0 + z * z / n
    c = (p + z * z / (2 * n)) / d
    h = z * math.sqrt(p * (1 - p) / n + z * z / (4 * n * n)) / d
    return (max(0.0, c - h), min(1.0, c + h))


def plan_units(units: list[tuple[int, int]], cost, world_size: int) -> list[list[tuple[int, int]]]:
    """Greedy longest-first assignment of (layer, block) units to ranks by cost(layer);
    deterministic (ties by unit order, then rank)."""
    order = sorted(range(len(units)), key=lambda i: (-cost(units[i][0]), i))
    load = [0.0] * world_size
    out: list[list[tuple[int, int]]] = [[] for _ in range(world_size)]
    for i in order:
        r = min(range(world_size), key=lambda j: (load[j], j))
        out[r].append(units[i])
        load[r] += cost(units[i][0])
    for o in out:
        o.sort()
    return out


@dataclass
class CampaignTally:
    """Per-layer counters (int64 [n_layers, len(FIELDS)]) plus the clean false-positive audit."""

    counters: np.ndarray
    clean_checks: int = 0
    clean_false_positive_checks: int = 0
    clean_false_positive_inferences: int = 0
    clean_inferences: int = 0
    records: dict = field(default_factory=dict)

    def total(self, name: str) -> int:
        return int(self.counters[:, FIELDS.index(name)].sum())

    def layer(self, i: int) -> dict:
        """Tallies of one layer, with the mean loss shift (corrupted - clean; injector.py:335-345)."""
        row = {name: int(v) for name, v in zip(FIELDS, self.counters[i])}
        n = row["injections"]
        row["loss_delta_sum"] = row.pop("loss_delta_fx") / LOSS_FX
        row["delta_loss"] = row["loss_delta_sum"] / n if n else 0.0
        return row

    @property
    def coverage(self) -> float:
        tp, fn = self.total("true_positives"), self.total("false_negatives")
        return tp / (tp + fn) if tp + fn else 1.0

    def by_group(self, groups: dict[str, list[int]]) -> dict:
        """Coverage per group of layers (e.g. the ViT roles): {name: [mismatches, TP, FN, coverage]}."""
        out = {}
        c = self.counters
        for name, idx in groups.items():
            mm = int(c[idx, FIELDS.index("mismatches")].sum())
            tp = int(c[idx, FIELDS.index("true_positives")].sum())
            fn = int(c[idx, FIELDS.index("false_negatives")].sum())
            out[name] = {"mismatches": mm, "true_positives": tp, "false_negatives": fn,
                         "coverage": tp / (tp + fn) if tp + fn else 1.0}
        return out

    def summary(self) -> dict:
        tp, fn = self.total("true_positives"), self.total("false_negatives")
        lo, hi = wilson_interval(tp, tp + fn)
        return {"injections": self.total("injections"), "skipped": self.total("skipped"),
                "mismatches": self.total("mismatches"), "true_positives": tp, "false_negatives": fn,
                "benign_detections": self.total("benign_detections"), "true_negatives": self.total("true_negatives"),
                "coverage_of_mismatches": self.coverage, "coverage_wilson95": [lo, hi],
                "clean_inferences": self.clean_inferences, "clean_checks": self.clean_checks,
                "clean_false_positive_checks": self.clean_false_positive_checks,
                "clean_false_positive_inferences": self.clean_false_positive_inferences,
                "false_flags_per_image": (self.clean_false_positive_checks / self.clean_inferences
                                          if self.clean_inferences else 0.0)}


@torch.no_grad()
def select_golden_images(model, teacher, make_batch, B: int, max_batches: int = 8) -> tuple[torch.Tensor, dict]:
    """Golden set of B images (profiler.select_golden, profiler.py:83-96): synthetic
    images labelled by a teacher (make_synthetic_dataset's teacher labelling,
    model.py:238-254) — here the same network at full precision (fp32 weights,
    binary32 GEMMs) — of which the deployed low-precision model keeps the ones it
    classifies correctly AND unambiguously: its top-2 logits more than two output
    ulps apart (a bf16 tie broken by argmax's index order is not a
    classification, and any perturbation would "mismatch" it).
    Returns (images [B, ...] on the device, stats)."""
    kept, seen, ties = [], 0, 0
    for _ in range(max_batches):
        imgs = make_batch()
        lab = teacher(imgs.to(teacher.dtype)).float().argmax(dim=1)
        lg = model(imgs)
        top2 = lg.float().topk(2, dim=1).values
        ulp = (top2[:, 0].abs() * 2.0 ** -(BF16_FIELDS[lg.dtype][0])).clamp_min(2.0 ** -24)
        clear = (top2[:, 0] - top2[:, 1]) > 2 * ulp
        ties += int((~clear).sum().item())
        ok = ((lab == lg.float().argmax(dim=1)) & clear).nonzero().flatten()
        kept.append(imgs[ok].clone())
        seen += imgs.shape[0]
        if sum(k.shape[0] for k in kept) >= B:
            break
    pool = torch.cat(kept)
    if pool.shape[0] < B:
        raise ValueError(f"only {pool.shape[0]} of {seen} images are classified like the teacher")
    return pool[:B].contiguous(), {"candidates": seen, "golden": int(pool.shape[0]),
                                   "golden_fraction": pool.shape[0] / seen, "near_ties_excluded": ties,
                                   "teacher": "same weights in fp32 (binary32 GEMMs)",
                                   "rule": "teacher label == model argmax and top-2 gap > 2 output ulps"}


def _flip16(bits: torch.Tensor, bit: torch.Tensor) -> torch.Tensor:
    """XOR one bit of 16-bit encodings (int16 storage), in int32 arithmetic."""
    v = (bits.to(torch.int32) & 0xFFFF) ^ torch.bitwise_left_shift(torch.ones_like(bit, dtype=torch.int32),
                                                                      bit.to(torch.int32))
    return (((v + 32768) & 0xFFFF) - 32768).to(torch.int16)


_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _uniform(seed: int, layer: int, k: np.ndarray, attempt: np.ndarray, draw: int) -> np.ndarray:
    """U[0, 1) as a function of (seed, layer, trial k, attempt, draw index): a SplitMix64
    finaliser over a mix of the counters (partition- and order-independent, vectorised)."""
    with np.errstate(over="ignore"):
        x = (np.uint64(seed & 0xFFFFFFFFFFFFFFFF) * np.uint64(0x9E3779B97F4A7C15)
             ^ np.uint64(layer) * np.uint64(0xC2B2AE3D27D4EB4F)
             ^ k * np.uint64(0x165667B19E3779F9) ^ attempt * np.uint64(0xD6E8FEB86659FD93)
             ^ np.uint64(draw) * np.uint64(0xFF51AFD7ED558CCD))
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


class ViTCampaign:
    """Output bit-flip campaign over the protected layers of a `ProtectedViT`.

    `images` [G, 3, H, W] on the device is the golden set (one forward batch);
    the clean pass records predictions, the per-layer clean range of the raw
    outputs (`gg_minmax`) and the prefix cache; `run` executes trial blocks of
    G trials per (layer, block)."""

    def __init__(self, model, images: torch.Tensor, *, seed: int = 0,
                 modes: tuple[str, ...] = ("fp_exponent_bit", "fp_mantissa_bit"), keep_records: bool = False):
        self.model, self.images, self.seed, self.modes = model, images, seed, modes
        self.G = images.shape[0]
        self.dev = images.device
        self.keep_records = keep_records
        self.fields = BF16_FIELDS[model.dtype]
        self.cache: dict = {}
        # the next block's sampling (clean output of its layer, retry gathers) runs on a side
        # stream while the previous block's suffix forward occupies the main one: its host
        # draws overlap the device work instead of waiting behind it
        self._side = torch.cuda.Stream(self.dev)
        self._y_layer, self._y = None, None
        with torch.no_grad():
            logits = model.forward(images, protect=True, cache=self.cache)
            self.clean_pred = logits.float().argmax(dim=1).clone()
            self.clean_loss = torch.nn.functional.cross_entropy(logits.float(), self.clean_pred, reduction="none")
            self.clean_flags = {i: self._image_flags(i) for i in range(model.cfg.n_layers)}
            res = model.buffers(self.G).results
            self._clean_nflag = dict(enumerate(torch.cat([res[i].nflag for i in range(model.cfg.n_layers)])
                                               .cpu().tolist()))
            self.ranges = {}
            self.raw = {}
            for i in range(model.cfg.n_layers):
                y = self._raw_output(i)
                rr = RunningRange(self.dev)
                rr.update(y)
                lo, hi, _ = rr.bounds()
                self.ranges[i] = (lo, hi)
        self._side.wait_stream(torch.cuda.current_stream(self.dev))  # the cache is read-only from here

    # ------------------------------------------------------------ helpers
    def _image_flags(self, i: int) -> torch.Tensor:
        res = self.model.buffers(self.G).results[i]
        rows = self.model.rows_per_image(i)
        return res.flags.view(self.G, rows).bool().any(dim=1)

    def _raw_output(self, i: int) -> torch.Tensor:
        """Clean raw (pre-activation) output of layer i from its cached input (unprotected launch)."""
        lin = self.model.layer(i)
        x = self.cache[i][1]
        y, _ = K.protected_gemm(x, lin.weight, lin.bias, protect=False, f32_mode=lin.f32_mode, w_split=lin.w_split)
        return y

    # ------------------------------------------------------------ sampling
    def _sample(self, layer: int, ks: np.ndarray, y: torch.Tensor):
        """Element / bit (or value) of each trial k (image k % G) by the reference's retry
        rules (injector.py:131-210: element, mode, then bit or value; no-op and range
        rejection; at most 64 attempts); elem -1 = skipped.  The draws are counter-based
        (`_uniform` of (seed, layer, k, attempt, draw)), vectorised over the block's trials
        and four attempts per round; the no-op / range tests run on the device.  Bit modes
        flip a bit of the stored encoding; "random_value" draws uniform(lo, hi) and stores
        it rounded to the output type.  Returns (elem, bit (-1 for value modes), mode
        index, value)."""
        rows = self.model.rows_per_image(layer)
        N = y.shape[1]
        n_elem = rows * N
        mant, exp = self.fields
        spans = {"fp_mantissa_bit": (0, mant), "fp_exponent_bit": (mant, mant + exp),
                 "fp_sign_bit": (mant + exp, mant + exp + 1)}
        for m in self.modes:
            if m not in spans and m != "random_value":
                raise ValueError(f"campaign mode {m!r} is not supported on the device engine")
        n = len(ks)
        elem = np.full(n, -1, dtype=np.int64)
        bit = np.full(n, -1, dtype=np.int64)
        mode_ix = np.zeros(n, dtype=np.int64)
        value = np.zeros(n, dtype=np.float64)
        pending = np.arange(n)
        lo, hi = self.ranges[layer]
        img = torch.from_numpy((ks % self.G).astype(np.int64)).to(self.dev)
        wide = y.element_size() == 2
        ybits = y.view(torch.int16) if wide else y.view(torch.int32)
        tries = 0
        span_lo = np.array([spans[m][0] if m in spans else 0 for m in self.modes], dtype=np.int64)
        span_w = np.array([spans[m][1] - spans[m][0] if m in spans else 0 for m in self.modes], dtype=np.int64)
        is_val = np.array([m == "random_value" for m in self.modes])
        while len(pending) and tries < MAX_RETRIES:
            r = min(ROUND, MAX_RETRIES - tries)
            # counter-based draws, vectorised over (trial, attempt): element, mode, then bit or value
            # -- the draw order of injector.py:169-186, each a function of (seed, layer, k, attempt)
            kk = ks[pending][:, None].astype(np.uint64)
            att = (tries + np.arange(r, dtype=np.uint64))[None, :]
            ce = np.minimum((_uniform(self.seed, layer, kk, att, 0) * n_elem).astype(np.int64), n_elem - 1)
            cm = np.minimum((_uniform(self.seed, layer, kk, att, 1) * len(self.modes)).astype(np.int64),
                            len(self.modes) - 1)
            u2 = _uniform(self.seed, layer, kk, att, 2)
            cb = np.where(is_val[cm], -1, span_lo[cm] + np.minimum((u2 * span_w[cm]).astype(np.int64),
                                                                 np.maximum(span_w[cm] - 1, 0)))
            cv = np.where(is_val[cm], lo + u2 * (hi - lo), 0.0)
            pe = torch.from_numpy(ce).to(self.dev)
            pb = torch.from_numpy(cb).to(self.dev)
            pimg = img[torch.from_numpy(pending).to(self.dev)].unsqueeze(1)
            grow = pimg * rows + pe // N
            gcol = pe % N
            orig = ybits[grow, gcol]
            isbit = pb >= 0
            sh = torch.bitwise_left_shift(torch.ones_like(pb, dtype=torch.int32), pb.clamp_min(0).to(torch.int32))
            flipped = _flip16(orig, pb.clamp_min(0)) if wide else orig ^ sh
            fv = torch.where(isbit, flipped.view(y.dtype).float(),
                             torch.from_numpy(cv).to(self.dev).to(y.dtype).float())  # value rounded like the store
            ov = orig.view(y.dtype).float()
            ok = (fv != ov) & (fv >= lo) & (fv <= hi)  # no-op and range rejection (injector.py:190-196)
            okh = ok.cpu().numpy()
            first = np.where(okh.any(axis=1), okh.argmax(axis=1), -1)
            done = first >= 0
            sel = pending[done]
            elem[sel] = ce[done, first[done]]
            bit[sel] = cb[done, first[done]]
            mode_ix[sel] = cm[done, first[done]]
            value[sel] = cv[done, first[done]]
            pending = pending[~done]
            tries += r
        return elem, bit, mode_ix, value

    # ----------------------------------------------------------------- run
    @torch.no_grad()
    def run_block(self, layer: int, block: int, counters: torch.Tensor) -> dict | None:
        """Trials k = block*G .. block*G + G - 1 of `layer`, one per image, folded into counters[layer]."""
        G = self.G
        ks = np.arange(block * G, (block + 1) * G, dtype=np.int64)
        main = torch.cuda.current_stream(self.dev)
        rows = self.model.rows_per_image(layer)
        with torch.cuda.stream(self._side):
            # every host <-> device copy of the sampling runs on the side stream: a pageable copy
            # waits for its stream, and on the main one that is the previous block's forward
            if self._y_layer != layer:  # the clean output of the layer, kept for its next blocks
                self._y, self._y_layer = self._raw_output(layer), layer
            y = self._y
            elem, bit, mode_ix, value = self._sample(layer, ks, y)
            ok = elem >= 0
            N = y.shape[1]
            img = ks % G
            grow = img * rows + np.where(ok, elem // N, 0)
            gcol = np.where(ok, elem % N, 0)
            inj = [K.Injection(row=int(r), col=int(c), bit=int(b)) if b >= 0 else
                   K.Injection(row=int(r), col=int(c), mode=L.GG_INJ_SET_VALUE, value=float(v))
                   for r, c, b, v, o in zip(grow, gcol, bit, value, ok) if o]
            inj_dev = K.injections_to_device(inj, self.dev)
            okd = torch.from_numpy(ok).to(self.dev)
        main.wait_stream(self._side)
        for t in (y, inj_dev, okd):
            t.record_stream(main)
        logits = self.model.resume(layer, self.cache, G, protect=True, injections={layer: inj_dev})
        lg = logits.float()
        pred = lg.argmax(dim=1)
        # loss shift against the clean prediction as label (the golden label, profiler.py:83-96)
        loss = torch.nn.functional.cross_entropy(lg, self.clean_pred, reduction="none")
        dl = torch.nan_to_num(loss - self.clean_loss, nan=LOSS_CLAMP, posinf=LOSS_CLAMP, neginf=-LOSS_CLAMP)
        dl_fx = torch.round(dl.clamp(-LOSS_CLAMP, LOSS_CLAMP).double() * LOSS_FX).to(torch.int64)
        mism = (pred != self.clean_pred) & okd
        det = self._image_flags(layer) & okd
        if not self.model.layer(layer).protected:
            det = torch.zeros_like(det)
        row = torch.stack([okd.sum(), mism.sum(), (mism & det).sum(), (mism & ~det).sum(), (~mism & det & okd).sum(),
                           (~mism & ~det & okd).sum(), (~okd).sum(), torch.where(okd, dl_fx, 0).sum()]).to(torch.int64)
        counters[layer] += row
        if not self.keep_records:
            return None
        orig_bits = y.view(torch.int16 if y.element_size() == 2 else torch.int32)[
            torch.from_numpy(grow).to(self.dev), torch.from_numpy(gcol).to(self.dev)]
        return {"layer": layer, "k": ks, "element": elem, "bit": bit, "mode": mode_ix, "value": value,
                "orig_bits": orig_bits.cpu().numpy(), "mismatch": mism.cpu().numpy(), "detected": det.cpu().numpy()}

    def run(self, n_blocks: int, layers=None, *, rank: int = 0, world_size: int = 1) -> CampaignTally:
        """n_blocks x G trials per layer; units shared over ranks by suffix cost, counters all-reduced (K5)."""
        nl = self.model.cfg.n_layers
        layers = list(range(nl)) if layers is None else list(layers)
        units = [(li, b) for li in layers for b in range(n_blocks)]
        mine = plan_units(units, lambda li: float(nl - li), world_size)[rank]
        counters = torch.zeros((nl, len(FIELDS)), dtype=torch.int64, device=self.dev)
        records = []
        for li, b in mine:
            rec = self.run_block(li, b, counters)
            if rec is not None:
                records.append(rec)
        Dd.reduce_counters(counters)
        audit = self.clean_counts()
        return CampaignTally(counters=counters.cpu().numpy(), records={"blocks": records}, **audit)

    def clean_counts(self) -> dict:
        """Clean false-positive audit of the golden batch: rows checked / flagged, images with any flag."""
        checks = fp_rows = 0
        any_flag = torch.zeros(self.G, dtype=torch.bool, device=self.dev)
        for i in range(self.model.cfg.n_layers):
            if not self.model.layer(i).protected:
                continue
            checks += self.G * self.model.rows_per_image(i)
            fp_rows += int(self._clean_nflag[i])
            any_flag |= self.clean_flags[i]
        return {"clean_checks": checks, "clean_false_positive_checks": fp_rows,
                "clean_false_positive_inferences": int(any_flag.sum().item()), "clean_inferences": self.G}
