"""Single-bit-flip fault injection: sampling, injected inference, campaigns.

Drop-in for ``gemmguard.injector`` (/root/reference/pkg/src/gemmguard/
injector.py).  The sampler reproduces the reference's draw order exactly
(injector.py:131-210), so the same (seed, layer, k), range profile and clean
trace give the same injected-error map.  Every GEMM of an injected inference
runs on the device through `model.run_layer`; campaigns can be sharded over
ranks (`run_campaign(..., rank=r, world=w)`) because every trial owns an RNG
stream derived from (seed, layer, k) (injector.py:451-452).

The batched, device-resident campaign engine (one trial per batch row,
in-epilogue injection, prefix reuse) is `paper_2310_03841_b200.campaign`.
"""

from __future__ import annotations

import csv
import io
import json
import math
import multiprocessing
from concurrent.futures import ProcessPoolExecutor
from dataclasses import dataclass, replace
from statistics import NormalDist

import numpy as np

from .errors import SamplingError
from .model import (
    ActivationTrace,
    ModelGraph,
    finish_layer_output,
    forward,
    loss_from_logits,
    output_dtype,
    prepare_layer_input,
    run_layer,
    working_array,
)
from .numerics import INT_DTYPES, Matrix2D, flip_bit, float_fields
from .profiler import GoldenSet, RangeProfile

__all__ = [
    "InjectionSpec",
    "InjectionRecord",
    "CampaignResult",
    "LOCATIONS",
    "BIT_MODES",
    "VALUE_MODES",
    "MAX_RETRIES",
    "sample_injection",
    "corrupted_value_for",
    "inject_forward",
    "injected_forward",
    "run_campaign",
    "margin_of_error",
    "default_modes",
    "bit_range",
    "injection_rng",
    "merge_campaigns",
]

LOCATIONS = ("input", "output", "weight")
BIT_MODES = ("int_bit", "fp_sign_bit", "fp_exponent_bit", "fp_mantissa_bit")
VALUE_MODES = ("random_value", "fixed_value")
MAX_RETRIES = 64  # injector.py:53


@dataclass(frozen=True)
class InjectionSpec:
    """One transient fault: layer, location, element, bit or value (injector.py:56-67)."""

    layer_index: int
    location: str
    element_index: int
    bit_index: int | None
    mode: str
    sample_id: int
    seed: int
    value: float | int | None = None


@dataclass
class InjectionRecord:
    """Outcome of one injected inference (injector.py:70-83)."""

    spec: InjectionSpec
    original_value: float
    corrupted_value: float
    golden_loss: float
    corrupted_loss: float
    golden_class: int
    corrupted_class: int
    mismatch: bool
    detected: bool | None = None
    detection_layer: int | None = None


def target_dtype(model: ModelGraph, location: str) -> str:
    """int models produce int32 outputs (injector.py:93-96)."""
    return "int32" if (location == "output" and model.is_integer) else model.dtype


def default_modes(model: ModelGraph, location: str = "output") -> tuple[str, ...]:
    """Exponent/mantissa flips for floats, any bit for ints (injector.py:86-90)."""
    return ("int_bit",) if target_dtype(model, location) in INT_DTYPES else ("fp_exponent_bit", "fp_mantissa_bit")


def bit_range(dtype: str, mode: str) -> tuple[int, int]:
    """Half-open bit interval a flip mode draws from (injector.py:99-111)."""
    if dtype in INT_DTYPES:
        if mode != "int_bit":
            raise ValueError(f"mode {mode!r} invalid for integer dtype {dtype}")
        return (0, 8 if dtype == "int8" else 32)
    mant, exp = float_fields(dtype)
    spans = {"fp_mantissa_bit": (0, mant), "fp_exponent_bit": (mant, mant + exp),
             "fp_sign_bit": (mant + exp, mant + exp + 1)}
    if mode not in spans:
        raise ValueError(f"mode {mode!r} invalid for floating dtype {dtype}")
    return spans[mode]


def _scalar(v, dtype: str):
    return int(v) if dtype in INT_DTYPES else float(v)


def _flipped(value, bit: int, dtype: str):
    return _scalar(flip_bit(value, bit, dtype), dtype)


def _target_values(model: ModelGraph, layer_index: int, location: str, trace: ActivationTrace) -> np.ndarray:
    if location == "output":
        return trace.outputs[layer_index].widened()
    if location == "input":
        return trace.inputs[layer_index].widened()
    if location == "weight":
        return model.layers[layer_index].weight.widened()
    raise ValueError(f"unknown injection location {location!r}")


def injection_rng(seed: int, layer_index: int, k: int) -> np.random.Generator:
    """Per-trial stream keyed by (seed, layer, k) (injector.py:451-452)."""
    return np.random.default_rng(np.random.SeedSequence((seed, layer_index, k)))


def sample_injection(
    model: ModelGraph,
    ranges: RangeProfile,
    golden: GoldenSet,
    rng: np.random.Generator,
    *,
    layer_index: int | None = None,
    sample_id: int | None = None,
    locations: tuple[str, ...] = ("output",),
    modes: tuple[str, ...] | None = None,
    seed: int = 0,
    clean_trace: ActivationTrace | None = None,
    max_retries: int = MAX_RETRIES,
) -> InjectionSpec:
    """Draw one range-respecting, value-changing fault (injector.py:131-210).

    Draw order: layer (if not given), sample (if not given), location, then
    per attempt element, mode, bit or value.  No-ops are redrawn; output
    faults must stay inside the profiled range; input/weight faults must stay
    finite.  Raises SamplingError after `max_retries` attempts.
    """
    if len(golden) == 0:
        raise ValueError("sample_injection requires a nonempty golden set")
    if layer_index is None:
        layer_index = int(rng.integers(len(model.layers)))
    if sample_id is None:
        sample_id = golden.sample_ids[int(rng.integers(len(golden)))]
    location = locations[int(rng.integers(len(locations)))]
    modes = modes if modes is not None else default_modes(model, location)
    dtype = target_dtype(model, location)
    if clean_trace is None:
        clean_trace = forward(model, golden.input_for(sample_id), golden.labels[sample_id], tap=[layer_index])
    values = _target_values(model, layer_index, location, clean_trace).ravel()
    lo, hi = ranges.bounds[layer_index]
    for _ in range(max_retries):
        element = int(rng.integers(values.size))
        mode = modes[int(rng.integers(len(modes)))]
        original = _scalar(values[element], dtype)
        bit = value = None
        if mode in BIT_MODES:
            b0, b1 = bit_range(dtype, mode)
            bit = int(rng.integers(b0, b1))
            corrupted = _flipped(original, bit, dtype)
        elif mode == "random_value":
            corrupted = int(rng.integers(int(lo), int(hi) + 1)) if dtype in INT_DTYPES else float(rng.uniform(lo, hi))
            value = corrupted
        else:
            raise ValueError(f"cannot sample mode {mode!r}")
        if corrupted == original:
            continue
        if location == "output":
            if not lo <= corrupted <= hi:
                continue
        elif isinstance(corrupted, float) and not math.isfinite(corrupted):
            continue
        return InjectionSpec(layer_index=layer_index, location=location, element_index=element, bit_index=bit,
                             mode=mode, sample_id=sample_id, seed=seed, value=value)
    raise SamplingError(f"layer {layer_index}: no in-range corruption found in {max_retries} attempts "
                        f"(range [{lo}, {hi}])")


def corrupted_value_for(spec: InjectionSpec, original: float, dtype: str) -> float:
    """Replacement value of a fault at its element (injector.py:213-221)."""
    if spec.mode in BIT_MODES:
        return _flipped(original, spec.bit_index, dtype)
    if spec.mode in VALUE_MODES:
        if spec.value is None:
            raise ValueError(f"{spec.mode} spec carries no value")
        return spec.value
    raise ValueError(f"unknown injection mode {spec.mode!r}")


def _check_element(spec: InjectionSpec, size: int) -> None:
    if not 0 <= spec.element_index < size:
        raise ValueError(f"element index {spec.element_index} out of range for size {size}")


def corrupt_operand(model: ModelGraph, layer, xin: np.ndarray, spec: InjectionSpec):
    """Scratch-copy corruption of a layer's input or weight (injector.py:247-263).

    Returns (xin, layer, original, corrupted); the model is never mutated."""
    if spec.location == "input":
        xin = np.array(xin, copy=True)
        flat = xin.reshape(-1)
        _check_element(spec, flat.size)
        orig = _scalar(flat[spec.element_index], model.dtype)
        bad = corrupted_value_for(spec, orig, model.dtype)
        flat[spec.element_index] = bad
        return xin, layer, orig, bad
    if spec.location == "weight":
        w = layer.weight.data.copy()
        flat = w.reshape(-1)
        _check_element(spec, flat.size)
        orig = _scalar(flat[spec.element_index], model.dtype)
        bad = corrupted_value_for(spec, orig, model.dtype)
        flat[spec.element_index] = bad
        return xin, replace(layer, weight=Matrix2D(w, model.dtype, _trusted=True)), orig, bad
    return xin, layer, math.nan, math.nan


def corrupt_output(model: ModelGraph, y: np.ndarray, spec: InjectionSpec):
    """Output fault on a copy of the raw GEMM output (injector.py:265-271)."""
    y = np.array(y, copy=True)
    flat = y.reshape(-1)
    _check_element(spec, flat.size)
    tag = output_dtype(model)
    orig = _scalar(flat[spec.element_index], tag)
    bad = corrupted_value_for(spec, orig, tag)
    flat[spec.element_index] = bad
    return y, orig, bad


def _trace(model, h, label, ins, outs) -> ActivationTrace:
    logits = h[0].astype(np.float64)
    return ActivationTrace(logits=logits, predicted_class=int(np.argmax(logits)),
                           loss=loss_from_logits(logits, label), label=label, inputs=ins, outputs=outs)


def injected_forward(model: ModelGraph, x: Matrix2D, label: int, spec: InjectionSpec,
                     tap: tuple[int, ...] = ()) -> tuple[ActivationTrace, float, float]:
    """Forward pass with one transient fault; returns (trace, original, corrupted) (injector.py:224-287)."""
    if not 0 <= spec.layer_index < len(model.layers):
        raise ValueError(f"layer index {spec.layer_index} out of range")
    tapped = frozenset(tap)
    h = working_array(model, x)
    ins, outs = {}, {}
    original = corrupted = math.nan
    for L in model.layers:
        xin = prepare_layer_input(model, L, h)
        run = L
        if L.index == spec.layer_index and spec.location in ("input", "weight"):
            xin, run, original, corrupted = corrupt_operand(model, L, xin, spec)
        y = np.asarray(run_layer(model, run, xin))
        if L.index == spec.layer_index and spec.location == "output":
            y, original, corrupted = corrupt_output(model, y, spec)
        if L.index in tapped:
            ins[L.index] = Matrix2D(xin, model.dtype, _trusted=True)
            outs[L.index] = Matrix2D(y, output_dtype(model), _trusted=True)
        h = finish_layer_output(model, L, y)
    return _trace(model, h, label, ins, outs), original, corrupted


def inject_forward(model: ModelGraph, x: Matrix2D, label: int, spec: InjectionSpec,
                   clean_trace: ActivationTrace | None = None) -> InjectionRecord:
    """One injection experiment and its record (injector.py:299-319)."""
    clean = clean_trace if clean_trace is not None else forward(model, x, label)
    t, orig, bad = injected_forward(model, x, label, spec)
    return InjectionRecord(spec=spec, original_value=orig, corrupted_value=bad, golden_loss=clean.loss,
                           corrupted_loss=t.loss, golden_class=clean.predicted_class,
                           corrupted_class=t.predicted_class, mismatch=t.predicted_class != clean.predicted_class)


# ------------------------------------------------------------------ campaigns
_CSV_COLUMNS = ["layer", "location", "element", "bit", "mode", "sample", "orig", "corrupt",
                "golden_loss", "corrupt_loss", "mismatch", "detected", "detection_layer"]


def _num(v) -> str:
    return str(v) if isinstance(v, int) else repr(float(v))


def _parse_num(s: str):
    try:
        return int(s)
    except ValueError:
        return float(s)


def _blank(v):
    return "" if v is None else v


@dataclass
class CampaignResult:
    """All records of a campaign plus per-layer tallies (injector.py:326-435)."""

    records: list[InjectionRecord]
    seed: int
    n_per_layer: int
    skipped: dict[int, int]

    def layer_tallies(self) -> dict[int, dict[str, float]]:
        out: dict[int, dict[str, float]] = {}
        for r in self.records:
            t = out.setdefault(r.spec.layer_index, {"injections": 0, "mismatches": 0, "loss_delta_sum": 0.0})
            t["injections"] += 1
            t["mismatches"] += int(r.mismatch)
            t["loss_delta_sum"] += r.corrupted_loss - r.golden_loss
        return out

    def to_csv(self) -> str:
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(_CSV_COLUMNS)
        for r in self.records:
            s = r.spec
            w.writerow([s.layer_index, s.location, s.element_index, _blank(s.bit_index), s.mode, s.sample_id,
                        _num(r.original_value), _num(r.corrupted_value), _num(r.golden_loss),
                        _num(r.corrupted_loss), int(r.mismatch),
                        "" if r.detected is None else int(r.detected), _blank(r.detection_layer)])
        return buf.getvalue()

    @classmethod
    def from_csv(cls, text: str, seed: int = 0, n_per_layer: int = 0) -> "CampaignResult":
        recs = []
        for row in csv.DictReader(io.StringIO(text)):
            bad = _parse_num(row["corrupt"])
            spec = InjectionSpec(layer_index=int(row["layer"]), location=row["location"],
                                 element_index=int(row["element"]),
                                 bit_index=None if row["bit"] == "" else int(row["bit"]), mode=row["mode"],
                                 sample_id=int(row["sample"]), seed=seed,
                                 value=bad if row["mode"] in VALUE_MODES else None)
            recs.append(InjectionRecord(
                spec=spec, original_value=_parse_num(row["orig"]), corrupted_value=bad,
                golden_loss=float(row["golden_loss"]), corrupted_loss=float(row["corrupt_loss"]),
                golden_class=-1, corrupted_class=-1, mismatch=bool(int(row["mismatch"])),
                detected=None if row["detected"] == "" else bool(int(row["detected"])),
                detection_layer=None if row["detection_layer"] == "" else int(row["detection_layer"])))
        return cls(records=recs, seed=seed, n_per_layer=n_per_layer, skipped={})

    def summary_json(self) -> str:
        doc = {"seed": self.seed, "n_per_layer": self.n_per_layer,
               "skipped": {str(k): v for k, v in sorted(self.skipped.items())},
               "layers": {str(k): {"injections": int(t["injections"]), "mismatches": int(t["mismatches"])}
                          for k, t in sorted(self.layer_tallies().items())}}
        return json.dumps(doc, indent=2, sort_keys=True)


def _layer_campaign(model, golden, ranges, layer_index, ks, modes, locations, seed):
    """Trials k in `ks` of one layer's stratum (injector.py:455-504)."""
    recs, skipped, cache = [], 0, {}
    for k in ks:
        rng = injection_rng(seed, layer_index, k)
        sid = golden.sample_ids[int(rng.integers(len(golden)))]
        if sid not in cache:
            cache[sid] = forward(model, golden.input_for(sid), golden.labels[sid], tap=[layer_index])
        clean = cache[sid]
        try:
            spec = sample_injection(model, ranges, golden, rng, layer_index=layer_index, sample_id=sid,
                                    locations=locations, modes=modes, seed=seed, clean_trace=clean)
        except SamplingError:
            skipped += 1
            continue
        recs.append(inject_forward(model, golden.input_for(sid), golden.labels[sid], spec, clean_trace=clean))
    return layer_index, recs, skipped


def run_campaign(model: ModelGraph, golden: GoldenSet, ranges: RangeProfile, n_per_layer: int, *,
                 modes: tuple[str, ...] | None = None, locations: tuple[str, ...] = ("output",), seed: int = 0,
                 workers: int = 1, rank: int = 0, world: int = 1) -> CampaignResult:
    """Stratified campaign, n_per_layer trials per layer (injector.py:507-565).

    `rank`/`world` keep the layers with index % world == rank (one shard per
    GPU; `merge_campaigns` restores the single-process result).  `workers` > 1
    runs layers in worker processes like the reference.  The result does not
    depend on workers or world: every trial owns its (seed, layer, k) stream.
    """
    if n_per_layer < 0:
        raise ValueError("n_per_layer must be >= 0")
    for loc in locations:
        if loc not in LOCATIONS:
            raise ValueError(f"unknown injection location {loc!r}")
    if n_per_layer == 0:
        return CampaignResult(records=[], seed=seed, n_per_layer=0, skipped={})
    mine = [li for li in range(len(model.layers)) if li % world == rank]
    if model.is_integer and tuple(locations) == ("output",):
        return _assemble(_batched_layer_campaigns(model, golden, ranges, mine, n_per_layer, modes, seed), seed,
                         n_per_layer)
    args = [(model, golden, ranges, li, range(n_per_layer), modes, locations, seed) for li in mine]
    if workers > 1:
        with ProcessPoolExecutor(max_workers=workers, mp_context=multiprocessing.get_context("spawn")) as pool:
            results = [f.result() for f in [pool.submit(_layer_campaign, *a) for a in args]]
    else:
        results = [_layer_campaign(*a) for a in args]
    return _assemble(results, seed, n_per_layer)


def _batched_layer_campaigns(model, golden, ranges, layers, n_per_layer, modes, seed):
    """Integer models, output faults: each layer's trials run as batched device forwards
    (guard.batched_injected_forwards, one fault per image in its own rows), drawn from the
    same per-trial streams as `_layer_campaign`; the records are identical."""
    from .guard import batched_injected_forwards, draw_trials

    tag = output_dtype(model)
    results, traces = [], {}
    for li in layers:
        drawn, traces = draw_trials(model, golden, ranges, li, range(n_per_layer), modes, seed, traces=traces)
        trials = [t for t in drawn if t[2] is not None]
        outs = batched_injected_forwards(model, golden, li, trials, protect=False)
        recs = []
        for (k, sid, spec), (_, pred, loss, _, _) in zip(trials, outs):
            clean = traces[sid]
            orig = _scalar(clean.outputs[li].widened().ravel()[spec.element_index], tag)
            recs.append(InjectionRecord(spec=spec, original_value=orig, corrupted_value=corrupted_value_for(spec, orig, tag),
                                        golden_loss=clean.loss, corrupted_loss=loss,
                                        golden_class=clean.predicted_class, corrupted_class=pred,
                                        mismatch=pred != clean.predicted_class))
        results.append((li, recs, len(drawn) - len(trials)))
    return results


def _assemble(results, seed: int, n_per_layer: int) -> CampaignResult:
    results = sorted(results, key=lambda r: r[0])
    return CampaignResult(records=[rec for _, recs, _ in results for rec in recs], seed=seed,
                          n_per_layer=n_per_layer, skipped={li: n for li, _, n in results if n})


def merge_campaigns(shards: list[CampaignResult]) -> CampaignResult:
    """Merge per-rank shards (disjoint layer sets) into the single-process result."""
    if not shards:
        raise ValueError("no shards to merge")
    per_layer: dict[int, list[InjectionRecord]] = {}
    for sh in shards:
        for rec in sh.records:
            per_layer.setdefault(rec.spec.layer_index, []).append(rec)
    skipped: dict[int, int] = {}
    for sh in shards:
        skipped.update(sh.skipped)
    layers = sorted(set(per_layer) | set(skipped))
    results = [(li, per_layer.get(li, []), skipped.get(li, 0)) for li in layers]
    return _assemble(results, shards[0].seed, shards[0].n_per_layer)


def margin_of_error(n: int, p: float, confidence: float) -> float:
    """z(confidence) * sqrt(p(1-p)/n) (injector.py:568-577)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if not 0.0 < p < 1.0:
        raise ValueError("p must lie in (0, 1)")
    if not 0.0 < confidence < 1.0:
        raise ValueError("confidence must lie in (0, 1)")
    return NormalDist().inv_cdf((1.0 + confidence) / 2.0) * math.sqrt(p * (1.0 - p) / n)
