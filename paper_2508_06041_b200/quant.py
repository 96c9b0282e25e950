"""Nested multi-scale store with device bitplanes (drop-in for ``dpq.quant``).

Host types and file formats mirror the reference
(``/root/reference/pkg/src/dpq/quant.py``): ``QuantizedLayer`` (quant.py:27-40),
``quantize_layer`` (quant.py:43-64, offline, numpy, bit-identical codes),
``BitPlaneStore`` (quant.py:102-110), ``pack_codes``/``unpack_codes``
(quant.py:123-135) and the ``.dpqs`` file (quant.py:140-181).

The numerics the decode path uses run on the GPU through libdpq_b200.so:
``gemv`` (quant.py:95-99) streams only planes 0..b-1 of the repacked
bitplanes, ``dequantize`` (quant.py:67-80) and ``delta_weights``
(quant.py:83-92) reconstruct from the same device planes.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import struct
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .model import KINDS, LayerId, ModelWeights, layer_ids

STORE_MAGIC = b"DPQS"
STORE_VERSION = 1


class QuantError(Exception):
    pass


class DeviceStore:
    """A dpq_store handle: device bitplanes of an ordered list of layers."""

    def __init__(self, layers, device=None):
        import torch
        dev = device if device is not None else _lib.torch_device()
        self.device = torch.device(dev)
        descs = (_lib.LayerDesc * len(layers))()
        keep = []
        for i, q in enumerate(layers):
            codes = np.ascontiguousarray(q.codes, dtype=np.uint16)
            lo = np.ascontiguousarray(q.lo, dtype=np.float32)
            hi = np.ascontiguousarray(q.hi, dtype=np.float32)
            keep += [codes, lo, hi]
            rows, cols = codes.shape
            descs[i] = _lib.LayerDesc(rows, cols, q.n_bits, q.b_min, 2, 0,
                                      codes.ctypes.data, lo.ctypes.data, hi.ctypes.data)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.call("dpq_store_create", self.device.index, len(layers), descs, C.byref(h))
        self.handle = h
        self.shapes = [tuple(q.codes.shape) for q in layers]
        self.bits = [(q.b_min, q.n_bits) for q in layers]
        self._fin = weakref.finalize(self, _destroy, "dpq_store_destroy", h.value)

    @staticmethod
    def from_device_codes(specs, device=None):
        """Build from device-resident codes: specs = [(codes_dev(uint16 or uint8 tensor),
        lo(np f32), hi(np f32), n_bits, b_min)] (large synthetic models)."""
        import torch
        self = DeviceStore.__new__(DeviceStore)
        self.device = torch.device(device if device is not None else _lib.torch_device())
        descs = (_lib.LayerDesc * len(specs))()
        keep = []
        for i, (codes, lo, hi, n_bits, b_min) in enumerate(specs):
            lo = np.ascontiguousarray(lo, dtype=np.float32)
            hi = np.ascontiguousarray(hi, dtype=np.float32)
            keep += [lo, hi]
            rows, cols = codes.shape
            descs[i] = _lib.LayerDesc(rows, cols, n_bits, b_min, codes.element_size(), 1,
                                      codes.data_ptr(), lo.ctypes.data, hi.ctypes.data)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.call("dpq_store_create", self.device.index, len(specs), descs, C.byref(h))
        self.handle = h
        self.shapes = [tuple(s[0].shape) for s in specs]
        self.bits = [(s[4], s[3]) for s in specs]
        self._fin = weakref.finalize(self, _destroy, "dpq_store_destroy", h.value)
        return self

    @staticmethod
    def empty(device=None):
        """A store filled layer by layer with ``append`` (streaming build: the
        caller frees each layer's codes before generating the next)."""
        import torch
        self = DeviceStore.__new__(DeviceStore)
        self.device = torch.device(device if device is not None else _lib.torch_device())
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.call("dpq_store_create", self.device.index, 0, None, C.byref(h))
        self.handle = h
        self.shapes, self.bits = [], []
        self._fin = weakref.finalize(self, _destroy, "dpq_store_destroy", h.value)
        return self

    def append(self, codes, lo, hi, n_bits: int, b_min: int):
        """Append one layer from device-resident codes (uint16 / uint8 / int16
        torch tensor); repacked into bitplanes on the device right away."""
        import torch
        lo = np.ascontiguousarray(lo, dtype=np.float32)
        hi = np.ascontiguousarray(hi, dtype=np.float32)
        rows, cols = codes.shape
        d = (_lib.LayerDesc * 1)()
        d[0] = _lib.LayerDesc(rows, cols, n_bits, b_min, codes.element_size(), 1, codes.data_ptr(),
                              lo.ctypes.data, hi.ctypes.data)
        with torch.cuda.device(self.device):
            _lib.call("dpq_store_append", self.handle, 1, d)
        self.shapes.append((rows, cols))
        self.bits.append((b_min, n_bits))

    def close(self):
        self._fin()

    def layer_bytes(self, i, b) -> int:
        out = C.c_int64()
        _lib.call("dpq_store_layer_bytes", self.handle, i, b, C.byref(out))
        return out.value

    def gemv(self, i, b, x, y=None):
        """y = W_b x on the device (torch float32 CUDA tensors)."""
        import torch
        rows, cols = self.shapes[i]
        x = x.to(device=self.device, dtype=torch.float32).contiguous()
        if y is None:
            y = torch.empty(rows, device=self.device, dtype=torch.float32)
        _lib.call("dpq_gemv", self.handle, i, b, C.c_void_p(x.data_ptr()),
                  C.c_void_p(y.data_ptr()), _lib.stream_ptr())
        return y

    def dequantize(self, i, b):
        import torch
        rows, cols = self.shapes[i]
        out = torch.empty((rows, cols), device=self.device, dtype=torch.float64)
        _lib.call("dpq_dequantize", self.handle, i, b, C.c_void_p(out.data_ptr()), _lib.stream_ptr())
        return out

    def exact_error(self, i, l, h, x) -> float:
        import torch
        x = x.to(device=self.device, dtype=torch.float32).contiguous()
        out = C.c_double()
        _lib.call("dpq_exact_error", self.handle, i, l, h, C.c_void_p(x.data_ptr()),
                  C.byref(out), _lib.stream_ptr())
        return float(out.value)


def _destroy(fn, ptr):
    try:
        if ptr:
            getattr(_lib.load(), fn)(C.c_void_p(ptr))
    except Exception:
        pass


@dataclass(eq=False)
class QuantizedLayer:
    codes: np.ndarray           # uint16 (rows, cols), each < 2**n_bits
    n_bits: int
    b_min: int
    lo: np.ndarray              # (rows,) float32
    hi: np.ndarray              # (rows,) float32
    _deq_cache: dict = field(default_factory=dict, repr=False)
    _dev: object = field(default=None, repr=False)      # (DeviceStore, index)

    @property
    def shape(self):
        return self.codes.shape

    def device_handle(self):
        """(DeviceStore, index) holding this layer's planes on the GPU."""
        if self._dev is None:
            self._dev = (DeviceStore([self]), 0)
        return self._dev


def quantize_layer(W: np.ndarray, n_bits: int, b_min: int) -> QuantizedLayer:
    """Per-output-channel affine codes floor((w-lo)*2^n/span) clipped to
    [0, 2^n-1]; span==0 rows get zero codes (offline, float64)."""
    if not (2 <= b_min <= n_bits <= 8):
        raise QuantError(f"need 2 <= b_min <= n_bits <= 8, got ({b_min}, {n_bits})")
    W = np.asarray(W, dtype=np.float64)
    if not np.all(np.isfinite(W)):
        raise QuantError("non-finite weights")
    lo, hi = W.min(axis=1), W.max(axis=1)
    span = hi - lo
    levels = 1 << n_bits
    with np.errstate(divide="ignore", invalid="ignore"):
        scaled = (W - lo[:, None]) * (levels / np.where(span == 0, 1.0, span))[:, None]
    codes = np.clip(np.floor(scaled), 0, levels - 1).astype(np.uint16)
    codes[span == 0, :] = 0
    return QuantizedLayer(codes, n_bits, b_min, lo.astype(np.float32), hi.astype(np.float32))


def _check_bits(layer, b):
    if not (layer.b_min <= b <= layer.n_bits):
        raise QuantError(f"bitwidth {b} outside [{layer.b_min}, {layer.n_bits}]")


def dequantize(layer: QuantizedLayer, b: int) -> np.ndarray:
    """Midpoint reconstruction of the b-bit variant, float64, computed on the
    device from the first b bitplanes (cached per b like the reference)."""
    _check_bits(layer, b)
    if b not in layer._deq_cache:
        ds, i = layer.device_handle()
        layer._deq_cache[b] = ds.dequantize(i, b).cpu().numpy()
    return layer._deq_cache[b]


def delta_weights(layer: QuantizedLayer, l: int, h: int) -> np.ndarray:
    """dequantize(h) - dequantize(l)."""
    if l >= h:
        raise QuantError(f"need l < h, got ({l}, {h})")
    key = ("delta", l, h)
    if key not in layer._deq_cache:
        layer._deq_cache[key] = dequantize(layer, h) - dequantize(layer, l)
    return layer._deq_cache[key]


def gemv(layer: QuantizedLayer, b: int, x):
    """W_b @ x on the device reading planes 0..b-1 only. numpy in -> float64
    numpy out (reference contract); a CUDA tensor in -> float32 CUDA tensor."""
    _check_bits(layer, b)
    shape_in = x.shape if hasattr(x, "shape") else np.asarray(x).shape
    if shape_in[-1] != layer.shape[1]:
        raise QuantError(f"gemv dimension mismatch: {shape_in[-1]} vs {layer.shape[1]}")
    ds, i = layer.device_handle()
    import torch
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return ds.gemv(i, b, x)
    xt = torch.as_tensor(np.asarray(x, dtype=np.float32), device=ds.device)
    return ds.gemv(i, b, xt).double().cpu().numpy()


@dataclass
class BitPlaneStore:
    layers: dict                # LayerId -> QuantizedLayer
    n_bits: int
    b_min: int
    config_hash: str
    _dev: object = field(default=None, repr=False, compare=False)

    def param_counts(self) -> dict:
        return {lid: int(np.prod(q.shape)) for lid, q in self.layers.items()}

    def ordered_ids(self):
        return sorted(self.layers, key=lambda l: (l.block, KINDS.index(l.kind)))

    def device_store(self) -> DeviceStore:
        """All layers in canonical (block, kind) order on the current GPU."""
        if self._dev is None:
            ids = self.ordered_ids()
            ds = DeviceStore([self.layers[l] for l in ids])
            for i, l in enumerate(ids):
                if self.layers[l]._dev is None:
                    self.layers[l]._dev = (ds, i)
            self._dev = ds
        return self._dev


def quantize_model(weights: ModelWeights, n_bits: int, b_min: int) -> BitPlaneStore:
    layers = {lid: quantize_layer(weights.linears[lid], n_bits, b_min)
              for lid in layer_ids(weights.config)}
    return BitPlaneStore(layers, n_bits, b_min, weights.config.hash())


# ---------------------------------------------------------------------------
# .dpqs file (reference format: quant.py:140-181)
# ---------------------------------------------------------------------------

def pack_codes(codes: np.ndarray, n_bits: int) -> bytes:
    """Code-major, LSB-first, n_bits per code, little-endian bytes."""
    flat = np.asarray(codes, dtype=np.uint16).reshape(-1)
    bits = ((flat[:, None] >> np.arange(n_bits)) & 1).astype(np.uint8)
    return np.packbits(bits.reshape(-1), bitorder="little").tobytes()


def unpack_codes(blob: bytes, n_bits: int, shape) -> np.ndarray:
    count = int(np.prod(shape))
    bits = np.unpackbits(np.frombuffer(blob, dtype=np.uint8), count=count * n_bits,
                         bitorder="little")
    w = 1 << np.arange(n_bits, dtype=np.uint16)
    return (bits.reshape(count, n_bits).astype(np.uint16) @ w).astype(np.uint16).reshape(shape)


def save_store(store: BitPlaneStore, path: str) -> None:
    with open(path, "wb") as f:
        f.write(STORE_MAGIC)
        f.write(struct.pack("<IBBBI", STORE_VERSION, store.n_bits, store.b_min, 0,
                            len(store.layers)))
        f.write(store.config_hash.encode("ascii"))
        for lid in store.ordered_ids():
            q = store.layers[lid]
            name = lid.name.encode("ascii")
            packed = pack_codes(q.codes, q.n_bits)
            f.write(struct.pack("<H", len(name)))
            f.write(name)
            f.write(struct.pack("<IIQ", q.shape[0], q.shape[1], len(packed)))
            f.write(np.ascontiguousarray(q.lo, dtype="<f4").tobytes())
            f.write(np.ascontiguousarray(q.hi, dtype="<f4").tobytes())
            f.write(packed)


def load_store(path: str) -> BitPlaneStore:
    with open(path, "rb") as f:
        if f.read(4) != STORE_MAGIC:
            raise QuantError("not a dpq store file")
        version, n_bits, b_min, bit_order, n_layers = struct.unpack("<IBBBI", f.read(11))
        if version != STORE_VERSION:
            raise QuantError(f"unsupported store version {version}")
        if bit_order != 0:
            raise QuantError("unsupported code bit order")
        config_hash = f.read(64).decode("ascii")
        layers = {}
        for _ in range(n_layers):
            (nlen,) = struct.unpack("<H", f.read(2))
            lid = LayerId.from_name(f.read(nlen).decode("ascii"))
            rows, cols, plen = struct.unpack("<IIQ", f.read(16))
            lo = np.frombuffer(f.read(4 * rows), dtype="<f4").copy()
            hi = np.frombuffer(f.read(4 * rows), dtype="<f4").copy()
            codes = unpack_codes(f.read(plen), n_bits, (rows, cols))
            layers[lid] = QuantizedLayer(codes, n_bits, b_min, lo, hi)
    return BitPlaneStore(layers, n_bits, b_min, config_hash)


def load_device_store(path: str, device=None) -> "DeviceBitPlaneStore":
    """Open a ``.dpqs`` file (quant.py:140-181) straight into device bitplanes.

    Same header checks and errors as ``load_store`` (quant.py:160-167), but each
    layer's packed code stream is uploaded as it lies on disk and repacked into
    MSB-first bitplanes by the device (``dpq_layer_desc.code_bytes = 0``): the
    host never materialises uint16 codes (numpy ``unpack_codes`` is the slow
    part of the reference loader at 7B+ sizes). The result quacks like a
    ``BitPlaneStore`` for the decode engine (``DeviceBitPlaneStore``).
    """
    with open(path, "rb") as f:
        if f.read(4) != STORE_MAGIC:
            raise QuantError("not a dpq store file")
        version, n_bits, b_min, bit_order, n_layers = struct.unpack("<IBBBI", f.read(11))
        if version != STORE_VERSION:
            raise QuantError(f"unsupported store version {version}")
        if bit_order != 0:
            raise QuantError("unsupported code bit order")
        config_hash = f.read(64).decode("ascii")
        entries = []
        for _ in range(n_layers):
            (nlen,) = struct.unpack("<H", f.read(2))
            lid = LayerId.from_name(f.read(nlen).decode("ascii"))
            rows, cols, plen = struct.unpack("<IIQ", f.read(16))
            if plen != (rows * cols * n_bits + 7) // 8:
                raise QuantError(f"{lid.name}: packed code length {plen} != rows*cols*n_bits/8")
            lo = np.frombuffer(f.read(4 * rows), dtype="<f4").astype(np.float32)
            hi = np.frombuffer(f.read(4 * rows), dtype="<f4").astype(np.float32)
            blob = np.frombuffer(f.read(plen), dtype=np.uint8)
            if blob.size != plen:
                raise QuantError(f"{lid.name}: truncated store file")
            entries.append((lid, rows, cols, lo, hi, blob))
    import torch
    dev = torch.device(device if device is not None else _lib.torch_device())
    # the engine indexes layers in (block, kind) order: 7*b + k
    entries.sort(key=lambda e: (e[0].block, KINDS.index(e[0].kind)))
    descs = (_lib.LayerDesc * len(entries))()
    for i, (lid, rows, cols, lo, hi, blob) in enumerate(entries):
        descs[i] = _lib.LayerDesc(rows, cols, n_bits, b_min, 0, 0, blob.ctypes.data,
                                  lo.ctypes.data, hi.ctypes.data)
    h = C.c_void_p()
    with torch.cuda.device(dev):
        _lib.call("dpq_store_create", dev.index, len(entries), descs, C.byref(h))
    ds = DeviceStore.__new__(DeviceStore)
    ds.device, ds.handle = dev, h
    ds.shapes = [(e[1], e[2]) for e in entries]
    ds.bits = [(b_min, n_bits)] * len(entries)
    ds._fin = weakref.finalize(ds, _destroy, "dpq_store_destroy", h.value)
    return DeviceBitPlaneStore(config_hash, n_bits, b_min,
                               {e[0]: (e[1], e[2]) for e in entries}, ds)


def file_hash(path: str) -> str:
    h = hashlib.sha256()
    with open(path, "rb") as f:
        for chunk in iter(lambda: f.read(1 << 20), b""):
            h.update(chunk)
    return h.hexdigest()


class _ShapeOnly:
    """Layer placeholder of a device-only store (codes live on the GPU)."""

    def __init__(self, shape, n_bits, b_min):
        self.shape = tuple(shape)
        self.n_bits, self.b_min = n_bits, b_min


class DeviceBitPlaneStore:
    """A BitPlaneStore whose codes exist only as device bitplanes (models too
    large to hold as host uint16 codes). Quacks like BitPlaneStore for the
    decode engine: config_hash, layers (shapes), param_counts, ordered_ids,
    device_store."""

    def __init__(self, config_hash, n_bits, b_min, shapes: dict, dstore: DeviceStore):
        self.config_hash = config_hash
        self.n_bits, self.b_min = n_bits, b_min
        self.layers = {lid: _ShapeOnly(s, n_bits, b_min) for lid, s in shapes.items()}
        self._dev = dstore

    def param_counts(self) -> dict:
        return {lid: int(np.prod(q.shape)) for lid, q in self.layers.items()}

    def ordered_ids(self):
        return sorted(self.layers, key=lambda l: (l.block, KINDS.index(l.kind)))

    def device_store(self) -> DeviceStore:
        return self._dev
