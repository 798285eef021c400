"""Relevance model containers + GPU scoring (mirror of nann.metric, metric.py:1-399).

The metric MLP is evaluated on the device by ``libgmpgr.so`` in numpy-einsum order,
so scores are bit-identical to the reference's ``relevance_batch`` (metric.py:150-154).
Projectors (feature -> embedding, metric.py:56-71) are input preparation, not the hot
path: they keep the reference's own numpy form so embeddings match byte for byte.
Weights are immutable once a model is used for inference (SPEC: model immutable).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import FileFormatError, InvalidArgumentError, WeightOverflowError

MODEL_MAGIC = b"NANN-MODEL"
MODEL_VERSION = 1
FP16_MAX = 65504.0
_ACTIVATIONS = ("relu", "identity")
_HEAD = "<IBBdIIII"  # version, fp16, activation, sigma, d_x, d_h, z_dim, n_layers


def _compute_dtype(arr: np.ndarray) -> np.dtype:
    # fp16 storage, fp32 arithmetic (metric.py:35-37)
    return np.dtype(np.float32) if arr.dtype == np.float16 else arr.dtype


@dataclass
class Projector:
    weight: np.ndarray  # (d_x, d_h)
    bias: np.ndarray    # (d_h,)

    @property
    def in_dim(self) -> int:
        return self.weight.shape[0]

    @property
    def out_dim(self) -> int:
        return self.weight.shape[1]


def project(projector: Projector, features: np.ndarray) -> np.ndarray:
    """Feature -> embedding (input preparation; reference form, metric.py:56-71)."""
    x = np.asarray(features)
    one = x.ndim == 1
    x = x[None, :] if one else x
    if x.shape[1] != projector.in_dim:
        raise InvalidArgumentError(
            f"feature dim {x.shape[1]} != projector input dim {projector.in_dim}")
    dt = _compute_dtype(projector.weight)
    y = np.einsum("ij,kj->ik", x.astype(dt, copy=False),
                  projector.weight.T.astype(dt, copy=False), optimize=False)
    y = y + projector.bias.astype(dt, copy=False)
    return y[0] if one else y


@dataclass(eq=False)
class MetricModel:
    """MLP over concat(h_u, h_v) -> Z heads -> attention dot (metric.py:74-99)."""

    layers: list
    attention: np.ndarray
    serendipity_sigma: float = 1.0
    activation: str = "relu"
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def precision(self) -> str:
        return "fp16" if self.layers[0][0].dtype == np.float16 else "fp32"

    @property
    def pair_dim(self) -> int:
        return self.layers[0][0].shape[1]

    @property
    def z_dim(self) -> int:
        return self.layers[-1][0].shape[0]

    def device_model(self, device: int | None = None) -> _lib.DeviceModel:
        """Cached device copy (processing-order weights, libgmpgr gr_model)."""
        device = _lib.current_device() if device is None else device
        h = self._dev.get(device)
        if h is None:
            if self.activation not in _ACTIVATIONS:
                raise InvalidArgumentError(f"unknown activation {self.activation!r}")
            for w, _ in self.layers:
                if w.dtype not in (np.float32, np.float16):
                    raise InvalidArgumentError(
                        "the device path computes in fp32: weights must be float32 or float16")
            h = _lib.DeviceModel(self.layers, self.attention, self.activation == "relu", device)
            self._dev[device] = h
        return h


@dataclass(eq=False)
class RelevanceModel:
    user_projector: Projector
    item_projector: Projector
    metric: MetricModel

    @property
    def precision(self) -> str:
        return self.metric.precision

    @property
    def d_x(self) -> int:
        return self.user_projector.in_dim

    @property
    def d_h(self) -> int:
        return self.user_projector.out_dim

    @property
    def z_dim(self) -> int:
        return self.metric.z_dim

    def user_embedding(self, features: np.ndarray) -> np.ndarray:
        return project(self.user_projector, features)

    def item_embeddings(self, features: np.ndarray) -> np.ndarray:
        return project(self.item_projector, features)

    def score(self, h_u: np.ndarray, h_v_batch: np.ndarray) -> np.ndarray:
        """One user against a batch of item embeddings (metric.py:222-226), on the GPU."""
        h_v_batch = np.atleast_2d(h_v_batch)
        return relevance_batch(self.metric, np.asarray(h_u)[None, :], h_v_batch,
                               broadcast_user=True).astype(np.float32)


def _metric_of(model) -> MetricModel:
    return model.metric if isinstance(model, RelevanceModel) else model


def relevance_batch(model, h_u: np.ndarray, h_v: np.ndarray, broadcast_user: bool = False):
    """Scalar relevance for n pairs (metric.py:150-154) computed by gr_score_pairs.

    Returns float32 scores bit-identical to the reference.  Raises NumericError on a
    non-finite final-layer value (metric.py:134-135).
    """
    metric = _metric_of(model)
    h_v = np.ascontiguousarray(np.atleast_2d(h_v), dtype=np.float32)
    h_u = np.ascontiguousarray(np.atleast_2d(h_u), dtype=np.float32)
    if not broadcast_user and h_u.shape != h_v.shape:
        raise InvalidArgumentError(f"embedding shapes differ: {h_u.shape} vs {h_v.shape}")
    if h_v.shape[1] * 2 != metric.pair_dim:
        raise InvalidArgumentError(f"embedding dim {h_v.shape[1]} != d_h {metric.pair_dim // 2}")
    n = h_v.shape[0]
    dm = metric.device_model()
    items = _lib.DeviceItems(h_v, dm.device)
    ids = np.arange(n, dtype=np.int64)
    uidx = None if broadcast_user else np.arange(n, dtype=np.int32)
    out = np.empty(n, dtype=np.float64)
    _lib.check(_lib.lib().gr_score_pairs(dm.h, items.h, _lib.ptr(h_u), h_u.shape[0],
                                         _lib.ptr(uidx), _lib.ptr(ids), n, _lib.ptr(out), 0, None))
    return out.astype(np.float32)


def relevance(model, h_u: np.ndarray, h_v: np.ndarray) -> float:
    return float(relevance_batch(model, np.asarray(h_u)[None, :], np.asarray(h_v)[None, :])[0])


def create_model(d_x: int, d_h: int, z_dim: int, hidden=(64, 64), seed: int = 0,
                 serendipity_sigma: float = 1.0, activation: str = "relu",
                 dtype=np.float32) -> RelevanceModel:
    """Random model with the reference's initialisation stream (metric.py:229-267):
    projectors N(0, 1/d_x), layers N(0, 1/fan_in), zero biases, attention 1/Z."""
    if activation not in _ACTIVATIONS:
        raise InvalidArgumentError(f"unknown activation {activation!r}")
    rng = np.random.default_rng(seed)
    projs = []
    for _ in range(2):
        w = (rng.normal(size=(d_x, d_h)) / np.sqrt(d_x)).astype(dtype)
        projs.append(Projector(w, np.zeros(d_h, dtype=dtype)))
    widths = [2 * d_h, *hidden, z_dim]
    layers = []
    for fan_in, fan_out in zip(widths[:-1], widths[1:]):
        w = (rng.normal(size=(fan_out, fan_in)) / np.sqrt(fan_in)).astype(dtype)
        layers.append((w, np.zeros(fan_out, dtype=dtype)))
    metric = MetricModel(layers, np.full(z_dim, 1.0 / z_dim, dtype=dtype), serendipity_sigma,
                         activation)
    return RelevanceModel(projs[0], projs[1], metric)


def _q16(a: np.ndarray, name: str) -> np.ndarray:
    if a.dtype == np.float16:
        return a.copy()
    if a.size and float(np.abs(a).max()) > FP16_MAX:
        raise WeightOverflowError(name, float(np.abs(a).max()))
    return a.astype(np.float16)


def quantize(model: RelevanceModel) -> RelevanceModel:
    """fp16 storage, fp32 inference (metric.py:280-307); idempotent."""
    up, ip, mm = model.user_projector, model.item_projector, model.metric
    return RelevanceModel(
        Projector(_q16(up.weight, "user_projector.weight"), _q16(up.bias, "user_projector.bias")),
        Projector(_q16(ip.weight, "item_projector.weight"), _q16(ip.bias, "item_projector.bias")),
        MetricModel([(_q16(w, f"mlp.{m}.weight"), _q16(b, f"mlp.{m}.bias"))
                     for m, (w, b) in enumerate(mm.layers)],
                    _q16(mm.attention, "attention"), mm.serendipity_sigma, mm.activation))


def save_model(model: RelevanceModel, path: str) -> None:
    """NANN-MODEL v1 writer (metric.py:310-341)."""
    fp16 = model.precision == "fp16"
    mm = model.metric
    out_dims = [w.shape[0] for w, _ in mm.layers]
    head = MODEL_MAGIC + struct.pack(_HEAD, MODEL_VERSION, int(fp16),
                                     _ACTIVATIONS.index(mm.activation), mm.serendipity_sigma,
                                     model.d_x, model.d_h, model.z_dim, len(mm.layers))
    head += struct.pack(f"<{len(out_dims)}I", *out_dims)
    blocks = [model.user_projector.weight, model.user_projector.bias,
              model.item_projector.weight, model.item_projector.bias]
    for w, b in mm.layers:
        blocks += [w, b]
    blocks.append(mm.attention)
    dt = "<f2" if fp16 else "<f4"
    with open(path, "wb") as f:
        f.write(head)
        for blk in blocks:
            f.write(np.ascontiguousarray(blk, dtype=dt).tobytes())


def load_model(path: str) -> RelevanceModel:
    """NANN-MODEL v1 reader (metric.py:344-399), same FileFormatError cases."""
    with open(path, "rb") as f:
        raw = f.read()
    if not raw.startswith(MODEL_MAGIC):
        raise FileFormatError("not a model file (bad magic)", path=path)
    off = len(MODEL_MAGIC)
    hs = struct.calcsize(_HEAD)
    if len(raw) < off + hs:
        raise FileFormatError("truncated model header", path=path)
    ver, fp16, act, sigma, d_x, d_h, z_dim, n_layers = struct.unpack_from(_HEAD, raw, off)
    if ver != MODEL_VERSION:
        raise FileFormatError(f"unsupported model version {ver}", path=path)
    if act >= len(_ACTIVATIONS):
        raise FileFormatError(f"unknown activation code {act}", path=path)
    off += hs
    if len(raw) < off + 4 * n_layers:
        raise FileFormatError("truncated layer dimension table", path=path)
    out_dims = struct.unpack_from(f"<{n_layers}I", raw, off)
    off += 4 * n_layers
    dt = np.dtype("<f2" if fp16 else "<f4")
    shapes = [(d_x, d_h), (d_h,), (d_x, d_h), (d_h,)]
    fan_in = 2 * d_h
    for d_out in out_dims:
        shapes += [(d_out, fan_in), (d_out,)]
        fan_in = d_out
    shapes.append((z_dim,))
    arrs = []
    for shp in shapes:
        cnt = int(np.prod(shp))
        nb = cnt * dt.itemsize
        if len(raw) < off + nb:
            raise FileFormatError(f"truncated weight block at byte {off}", path=path)
        arrs.append(np.frombuffer(raw, dtype=dt, count=cnt, offset=off).reshape(shp).copy())
        off += nb
    if off != len(raw):
        raise FileFormatError(f"{len(raw) - off} trailing bytes", path=path)
    if out_dims and out_dims[-1] != z_dim:
        raise FileFormatError("final layer width != z_dim", path=path)
    it = iter(arrs)
    up = Projector(next(it), next(it))
    ip = Projector(next(it), next(it))
    layers = [(next(it), next(it)) for _ in range(n_layers)]
    return RelevanceModel(up, ip, MetricModel(layers, next(it), sigma, _ACTIVATIONS[act]))
