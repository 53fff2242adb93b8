"""The reference's "ALBT" v1 weight container, read straight into device memory
(format: /root/reference/pkg/src/gemmguard/weights_io.py:1-7).

Layout (little-endian): b"ALBT", u32 version = 1, u32 tensor count; per tensor
u16 name length, UTF-8 name, u8 dtype tag {0 f64, 1 f32, 2 f16, 3 i8, 4 i32},
u8 rank, rank x u32 dims, row-major payload.  `graph.meta` (i32 x 6: tokens,
classes, input dim, model dtype tag, seed low / high word) describes the graph;
layers are `layer{index:03d}.{kind}.{weight|bias}` with the weight stored as the
reference's Wt [in, out].

`load_device` parses the container once, copies every payload into one pinned
host arena and moves it to the device in a single transfer; each layer's
weight is then transposed on the device into the torch layout [out, in] that
K1 reads, and its offline checksum (K2) is taken there.  `load_model` returns
the reference's `ModelGraph` (host) for the drop-in API; `save` writes the
same bytes as the reference's `save_weights`.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from . import kernels as K
from .errors import WeightFormatError
from .model import LayerSpec, ModelGraph
from .numerics import Matrix2D

__all__ = ["MAGIC", "VERSION", "read_tensors", "load_model", "load_device", "save", "DeviceWeights"]

MAGIC = b"ALBT"
VERSION = 1
_NP = {0: "<f8", 1: "<f4", 2: "<f2", 3: "<i1", 4: "<i4"}
_MODEL_DTYPE = {0: "binary64", 1: "binary32", 2: "binary16-emulated", 3: "int8", 4: "int32"}
_TAG = {v: k for k, v in _MODEL_DTYPE.items()}


def read_tensors(blob: bytes) -> dict[str, tuple[int, np.ndarray]]:
    """name -> (dtype tag, array view into `blob`) with the reference's format checks."""
    if blob[:4] != MAGIC:
        raise WeightFormatError("bad magic")
    if len(blob) < 12:
        raise WeightFormatError("truncated container while reading header")
    version, count = struct.unpack_from("<II", blob, 4)
    if version != VERSION:
        raise WeightFormatError(f"version mismatch: got {version}, expected {VERSION}")
    off, out = 12, {}
    for _ in range(count):
        if off + 2 > len(blob):
            raise WeightFormatError("truncated container while reading tensor name length")
        (n,) = struct.unpack_from("<H", blob, off)
        name = blob[off + 2:off + 2 + n].decode("utf-8")
        off += 2 + n
        if off + 2 > len(blob):
            raise WeightFormatError(f"truncated container while reading tensor {name} header")
        tag, rank = struct.unpack_from("<BB", blob, off)
        off += 2
        if tag not in _NP:
            raise WeightFormatError(f"tensor {name}: unknown dtype tag {tag}")
        if rank > 2:
            raise WeightFormatError(f"tensor {name}: unsupported rank {rank}")
        dims = struct.unpack_from(f"<{rank}I", blob, off)
        off += 4 * rank
        dt = np.dtype(_NP[tag])
        size = int(np.prod(dims, dtype=np.int64)) * dt.itemsize
        if off + size > len(blob):
            raise WeightFormatError(f"truncated container while reading tensor {name} payload")
        out[name] = (tag, np.frombuffer(blob, dtype=dt, count=size // dt.itemsize, offset=off).reshape(dims))
        off += size
    return out


def _graph(tensors) -> tuple[dict, list[tuple[int, str, np.ndarray, np.ndarray]]]:
    if "graph.meta" not in tensors:
        raise WeightFormatError("missing graph.meta tensor")
    meta = tensors["graph.meta"][1].astype(np.int64)
    dtype = _MODEL_DTYPE.get(int(meta[3]))
    if dtype is None:
        raise WeightFormatError(f"graph.meta: unknown model dtype tag {int(meta[3])}")
    info = {"tokens": int(meta[0]), "classes": int(meta[1]), "input_dim": int(meta[2]), "dtype": dtype,
            "seed": (int(meta[4]) & 0xFFFFFFFF) | ((int(meta[5]) & 0xFFFFFFFF) << 32)}
    layers: dict[int, dict] = {}
    for name, (_, arr) in tensors.items():
        if name == "graph.meta":
            continue
        parts = name.split(".")
        if len(parts) != 3 or not parts[0].startswith("layer") or not parts[0][5:].isdigit():
            raise WeightFormatError(f"unrecognized tensor name {name!r}")
        entry = layers.setdefault(int(parts[0][5:]), {"kind": parts[1]})
        entry[parts[2]] = arr
    out = []
    for i in sorted(layers):
        e = layers[i]
        if "weight" not in e or "bias" not in e:
            raise WeightFormatError(f"layer {i}: missing weight or bias tensor")
        if e["weight"].ndim != 2 or e["bias"].ndim != 1:
            raise WeightFormatError(f"layer {i}: bad tensor ranks")
        out.append((i, e["kind"], e["weight"], e["bias"]))
    return info, out


def load_model(path) -> ModelGraph:
    """The container as the reference's ModelGraph (weights_io.load_weights' result)."""
    with open(path, "rb") as f:
        info, layers = _graph(read_tensors(f.read()))
    dt = info["dtype"]
    integer = dt in ("int8", "int32")
    specs = []
    for i, kind, w, b in layers:
        wv = w.astype(np.float64) if dt == "binary16-emulated" else w
        bv = b.astype(np.int32) if integer else b.astype(np.float64)
        act = ("relu" if integer else "gelu") if kind == "mlp_fc1" else "none"
        specs.append(LayerSpec(index=i, name=f"layer{i:03d}.{kind}", kind=kind, in_dim=w.shape[0], out_dim=w.shape[1],
                               tokens=1 if kind == "head" else info["tokens"], weight=Matrix2D(wv, dt), bias=bv,
                               activation=act, normalize_before=(not integer) and kind in ("qkv", "mlp_fc1", "head")))
    return ModelGraph(layers=specs, num_classes=info["classes"], input_dim=info["input_dim"], tokens=info["tokens"],
                      dtype=dt, seed=info["seed"])


@dataclass
class DeviceWeights:
    """Device copies of a container: per layer the weight in torch layout [out, in], the bias,
    and the offline checksum (K2) in the layer's checksum precision."""

    info: dict
    weights: dict[int, torch.Tensor]
    biases: dict[int, torch.Tensor]
    w_sum: dict[int, torch.Tensor]
    bias_sum: dict[int, float | int]


def load_device(path, device="cuda", precision: int = L.GG_P_F64) -> DeviceWeights:
    """Parse once, one pinned host -> device copy of every payload, device transposes and K2."""
    with open(path, "rb") as f:
        blob = f.read()
    info, layers = _graph(read_tensors(blob))
    dev = torch.device(device)
    host = torch.from_numpy(np.frombuffer(blob, dtype=np.uint8).copy()).pin_memory()
    arena = host.to(dev, non_blocking=True)  # the whole container in one transfer
    base = np.frombuffer(blob, dtype=np.uint8).ctypes.data
    integer = info["dtype"] in ("int8", "int32")
    tdt = {"binary64": torch.float64, "binary32": torch.float32, "binary16-emulated": torch.float16,
           "int8": torch.int8, "int32": torch.int32}[info["dtype"]]

    def view(arr, dt):  # payloads are packed unaligned: a device copy per tensor realigns it
        off = arr.ctypes.data - base
        return arena[off:off + arr.nbytes].clone().view(dt).view(arr.shape)

    weights, biases, w_sum, bias_sum = {}, {}, {}, {}
    for i, _, w, b in layers:
        wt = view(w, tdt)                      # Wt [in, out] as stored
        weights[i] = wt.t().contiguous()       # [out, in]: K1's K-major operand
        bt = view(b, torch.int32 if integer else {4: torch.float32, 8: torch.float64, 2: torch.float16}[b.itemsize])
        biases[i] = bt.to(torch.int32 if integer else torch.float32)
        ws, bs = K.offline_checksum(wt, bt.to(torch.int64 if integer else torch.float64),
                                    L.GG_P_I64 if integer else precision, layout=1)
        w_sum[i] = ws
        bias_sum[i] = int(bs.item()) if integer else float(bs.item())
    return DeviceWeights(info, weights, biases, w_sum, bias_sum)


def save(path, model: ModelGraph) -> None:
    """The reference's byte layout (weights_io.save_weights)."""
    seed = int(model.seed) & 0xFFFFFFFFFFFFFFFF
    meta = np.array([model.tokens, model.num_classes, model.input_dim, _TAG[model.dtype],
                     np.uint32(seed & 0xFFFFFFFF).view(np.int32), np.uint32(seed >> 32).view(np.int32)],
                    dtype=np.int32)
    chunks = [MAGIC, struct.pack("<II", VERSION, 2 * len(model.layers) + 1)]

    def tensor(name, arr, tag):
        enc = name.encode("utf-8")
        arr = np.ascontiguousarray(np.asarray(arr).astype(_NP[tag]))
        chunks.append(struct.pack("<H", len(enc)) + enc + struct.pack("<BB", tag, arr.ndim) +
                      struct.pack(f"<{arr.ndim}I", *arr.shape) + arr.tobytes())

    tensor("graph.meta", meta, 4)
    integer = model.dtype in ("int8", "int32")
    for ly in model.layers:
        base = f"layer{ly.index:03d}.{ly.kind}"
        tensor(f"{base}.weight", ly.weight.data, _TAG[model.dtype])
        tensor(f"{base}.bias", ly.bias, 4 if integer else _TAG[model.dtype])
    with open(path, "wb") as f:
        f.write(b"".join(chunks))
