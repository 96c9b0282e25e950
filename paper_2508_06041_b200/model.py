"""Model-side types for the decode path (host).

Mirrors the reference ``dpq.model`` surface the hot path consumes
(``/root/reference/pkg/src/dpq/model.py``): ``ModelConfig`` (model.py:45-81),
``LayerId`` (model.py:22-42), ``layer_ids``/``layer_shape`` (model.py:84-94),
``ModelWeights`` (model.py:97-110), ``init_model`` (model.py:113-128) and the
weight manifest I/O (model.py:139-193). One extension: ``n_kv_heads`` (GQA,
Llama-3-8B / Llama-2-70B shapes); it is left out of ``to_dict``/``hash`` when
equal to ``n_heads`` so MHA configs hash exactly like the reference's.

The numerics of the model live on the device (``runtime.DecodeEngine``);
this module is plain host data plumbing.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass

import numpy as np

KINDS = ("q", "k", "v", "o", "up", "gate", "down")
RESIDUAL_FED_KINDS = frozenset({"q", "k", "v", "up"})
ROPE_BASE = 10000.0


@dataclass(frozen=True)
class LayerId:
    """One linear layer: (block index, kind). Name ``block{b}.{kind}``."""

    block: int
    kind: str

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown layer kind {self.kind!r}")

    @property
    def name(self) -> str:
        return f"block{self.block}.{self.kind}"

    @property
    def residual_fed(self) -> bool:
        return self.kind in RESIDUAL_FED_KINDS

    @staticmethod
    def from_name(name: str) -> "LayerId":
        blk, kind = name.split(".")
        return LayerId(int(blk.removeprefix("block")), kind)

    def __hash__(self):
        return hash((self.block, self.kind))

    def __eq__(self, other):
        # interoperate with any LayerId-like object (e.g. the reference's)
        try:
            return (self.block, self.kind) == (other.block, other.kind)
        except AttributeError:
            return NotImplemented


@dataclass(frozen=True)
class ModelConfig:
    n_blocks: int
    d_model: int
    n_heads: int
    d_ff: int
    vocab: int = 256
    seq_cap: int = 1024
    norm_eps: float = 1e-6
    n_kv_heads: int | None = None

    def __post_init__(self):
        for f in ("n_blocks", "d_model", "n_heads", "d_ff", "vocab", "seq_cap"):
            if getattr(self, f) < 1:
                raise ValueError(f"{f} must be >= 1")
        if self.d_model % self.n_heads != 0:
            raise ValueError("d_model must be divisible by n_heads")
        if self.norm_eps <= 0:
            raise ValueError("norm_eps must be positive")
        if self.n_kv_heads is not None:
            if self.n_kv_heads < 1 or self.n_heads % self.n_kv_heads != 0:
                raise ValueError("n_heads must be a multiple of n_kv_heads")
            if self.n_kv_heads == self.n_heads:
                object.__setattr__(self, "n_kv_heads", None)

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    @property
    def kv_heads(self) -> int:
        return self.n_kv_heads or self.n_heads

    @property
    def d_kv(self) -> int:
        return self.kv_heads * self.head_dim

    def to_dict(self) -> dict:
        d = {"n_blocks": self.n_blocks, "d_model": self.d_model,
             "n_heads": self.n_heads, "d_ff": self.d_ff, "vocab": self.vocab,
             "seq_cap": self.seq_cap, "norm_eps": self.norm_eps}
        if self.n_kv_heads is not None:
            d["n_kv_heads"] = self.n_kv_heads
        return d

    @staticmethod
    def from_dict(d: dict) -> "ModelConfig":
        return ModelConfig(**d)

    def hash(self) -> str:
        return hashlib.sha256(json.dumps(self.to_dict(), sort_keys=True).encode()).hexdigest()


def rope_tables(n_pos: int, head_dim: int):
    """Half-split RoPE tables (reference model.py:206-212): cos, sin of shape
    (n_pos, head_dim // 2), float64; (None, None) when head_dim < 2."""
    half = head_dim // 2
    if half == 0:
        return None, None
    inv_freq = ROPE_BASE ** (-np.arange(half, dtype=np.float64) * 2.0 / head_dim)
    angles = np.arange(n_pos, dtype=np.float64)[:, None] * inv_freq[None, :]
    return np.cos(angles), np.sin(angles)


def layer_ids(config: ModelConfig) -> list:
    """Canonical order: blocks ascending, kinds q,k,v,o,up,gate,down."""
    return [LayerId(b, k) for b in range(config.n_blocks) for k in KINDS]


def layer_shape(config: ModelConfig, lid) -> tuple:
    d, f, dkv = config.d_model, config.d_ff, config.d_kv
    return {"q": (d, d), "k": (dkv, d), "v": (dkv, d), "o": (d, d),
            "up": (f, d), "gate": (f, d), "down": (d, f)}[lid.kind]


@dataclass
class ModelWeights:
    config: ModelConfig
    embed: np.ndarray       # (vocab, d) float32
    lm_head: np.ndarray     # (vocab, d) float32; logits = lm_head @ norm(x)
    linears: dict           # LayerId -> float32 (rows, cols); may be empty
                            # when the model only exists as a quantized store

    def checksum(self) -> str:
        h = hashlib.sha256()
        h.update(self.embed.tobytes())
        h.update(self.lm_head.tobytes())
        for lid in layer_ids(self.config):
            h.update(self.linears[lid].tobytes())
        return h.hexdigest()


def init_model(seed: int, config: ModelConfig) -> ModelWeights:
    """Seeded random init drawing the same stream as the reference, so equal
    (seed, config) give bit-identical float32 weights and store hashes."""
    rng = np.random.default_rng(seed)
    d = config.d_model
    embed = rng.normal(0.0, 1.0, (config.vocab, d)).astype(np.float32)
    lm_head = (rng.normal(0.0, 1.0, (config.vocab, d)) * (0.1 / np.sqrt(d))).astype(np.float32)
    linears = {}
    for lid in layer_ids(config):
        rows, cols = layer_shape(config, lid)
        linears[lid] = rng.normal(0.0, 1.0 / np.sqrt(cols), (rows, cols)).astype(np.float32)
    return ModelWeights(config, embed, lm_head, linears)


class WeightFormatError(Exception):
    pass


WEIGHTS_FORMAT = "dpq-weights-v1"


def export_weights(weights: ModelWeights, manifest_path: str) -> None:
    """JSON manifest + one flat little-endian float32 file (same format as
    the reference's model.py:139-156)."""
    bin_path = str(manifest_path) + ".bin"
    tensors = [("embed", weights.embed), ("lm_head", weights.lm_head)]
    tensors += [(lid.name, weights.linears[lid]) for lid in layer_ids(weights.config)]
    entries, off = [], 0
    with open(bin_path, "wb") as f:
        for name, arr in tensors:
            arr = np.ascontiguousarray(arr, dtype="<f4")
            f.write(arr.tobytes())
            entries.append({"name": name, "shape": list(arr.shape), "dtype": "float32",
                            "offset": off, "nbytes": arr.nbytes})
            off += arr.nbytes
    with open(manifest_path, "w") as f:
        json.dump({"format": WEIGHTS_FORMAT, "config": weights.config.to_dict(),
                   "data_file": bin_path.rsplit("/", 1)[-1], "tensors": entries}, f, indent=1)


def load_weights(manifest_path: str) -> ModelWeights:
    with open(manifest_path) as f:
        man = json.load(f)
    if man.get("format") != WEIGHTS_FORMAT:
        raise WeightFormatError("not a dpq weight manifest")
    config = ModelConfig.from_dict(man["config"])
    parts = str(manifest_path).rsplit("/", 1)
    bin_path = parts[0] + "/" + man["data_file"] if len(parts) > 1 else man["data_file"]
    raw = np.memmap(bin_path, dtype=np.uint8, mode="r")
    by_name = {}
    for e in man["tensors"]:
        end = e["offset"] + e["nbytes"]
        if end > len(raw):
            raise IOError(f"weight file truncated: tensor {e['name']} needs bytes "
                          f"up to {end}, file has {len(raw)}")
        by_name[e["name"]] = np.frombuffer(raw[e["offset"]:end].tobytes(),
                                           dtype="<f4").reshape(e["shape"])

    def expect(name, shape):
        if name not in by_name:
            raise WeightFormatError(f"missing tensor entry: {name}")
        if tuple(by_name[name].shape) != tuple(shape):
            raise WeightFormatError(f"shape mismatch for tensor {name}: manifest "
                                    f"{by_name[name].shape}, config requires {tuple(shape)}")
        return by_name[name]

    embed = expect("embed", (config.vocab, config.d_model))
    lm_head = expect("lm_head", (config.vocab, config.d_model))
    linears = {lid: expect(lid.name, layer_shape(config, lid)) for lid in layer_ids(config)}
    return ModelWeights(config, embed, lm_head, linears)


def forward(weights, tokens, provider=None, want_tape: bool = False):
    """model.py:286-345 (fp64 device graph: graph.forward)."""
    from . import graph
    return graph.forward(weights, tokens, provider, want_tape)


def backward(weights, tokens, provider=None):
    """model.py:382-460 (fp64 device graph: graph.backward)."""
    from . import graph
    return graph.backward(weights, tokens, provider)


def teacher_forced_loss(weights, tokens, provider=None):
    """model.py:363-372 (graph.teacher_forced_loss)."""
    from . import graph
    return graph.teacher_forced_loss(weights, tokens, provider)
