"""Decoder checkpoints in the reference's LIPSUBCKPT1 format, so trained reference models
drive the B200 solver (restates proj/src/net.cpp:259-353):

    "LIPSUBCKPT1\\n" | u64 little-endian header length | JSON header
    {"format": "lipsub-checkpoint", "r", "n", "decoder": [{"rows", "cols", "act"}...],
     "encoder": [...]} | little-endian f64 blob: per decoder layer W row-major then b, per
    encoder layer the same, then norm_shift (n) and norm_scale (n).

Errors follow the reference: unreadable / bad magic / truncated -> RuntimeError
(std::runtime_error); shape or activation problems -> ValueError (std::invalid_argument).
The encoder (training-time only) is kept on `model.encoder` and not used by the solver."""
from __future__ import annotations

import json
import struct
from typing import List

import numpy as np

from .lipsub import Activation, Layer, SubspaceModel, activation_from_string

MAGIC = b"LIPSUBCKPT1\n"
_NAMES = {Activation.Identity: "identity", Activation.Silu: "silu", Activation.Tanh: "tanh",
          Activation.Elu: "elu"}  # 'elu': BASELINE.json extension


def _meta(layers: List[Layer]):
    return [{"rows": int(l.W.shape[0]), "cols": int(l.W.shape[1]), "act": _NAMES[Activation(l.act)]}
            for l in layers]


def save_checkpoint(model: SubspaceModel, path: str) -> None:
    """reference save_checkpoint (net.cpp:280-308)."""
    model.validate()
    encoder = getattr(model, "encoder", [])
    header = {"format": "lipsub-checkpoint", "r": int(model.r), "n": int(model.n),
              "decoder": _meta(model.decoder), "encoder": _meta(encoder)}
    hs = json.dumps(header, separators=(",", ":")).encode()
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<Q", len(hs)))
        f.write(hs)
        for l in list(model.decoder) + list(encoder):
            f.write(np.ascontiguousarray(l.W, "<f8").tobytes())  # row-major
            f.write(np.ascontiguousarray(l.b, "<f8").tobytes())
        f.write(np.ascontiguousarray(model.norm_shift, "<f8").tobytes())
        f.write(np.ascontiguousarray(model.norm_scale, "<f8").tobytes())


def load_checkpoint(path: str) -> SubspaceModel:
    """reference load_checkpoint (net.cpp:310-353)."""
    try:
        f = open(path, "rb")
    except OSError:
        raise RuntimeError(f"checkpoint: cannot open '{path}'")
    with f:
        data = f.read()
    if data[:len(MAGIC)] != MAGIC:
        raise RuntimeError(f"checkpoint: bad magic in '{path}'")
    pos = len(MAGIC)
    if len(data) < pos + 8:
        raise RuntimeError("checkpoint: truncated header")
    (hlen,) = struct.unpack_from("<Q", data, pos)
    pos += 8
    if len(data) < pos + hlen:
        raise RuntimeError("checkpoint: truncated header")
    header = json.loads(data[pos:pos + hlen].decode())
    pos += hlen

    def blob(count: int) -> np.ndarray:
        nonlocal pos
        nbytes = 8 * count
        if len(data) < pos + nbytes:
            raise RuntimeError("checkpoint: truncated weight blob")
        out = np.frombuffer(data, "<f8", count, pos).astype(np.float64)
        pos += nbytes
        return out

    def layers(meta) -> List[Layer]:
        out = []
        for lm in meta:
            rows, cols = int(lm["rows"]), int(lm["cols"])
            act = activation_from_string(lm["act"])
            W = blob(rows * cols).reshape(rows, cols)
            b = blob(rows)
            out.append(Layer(W, b, act))
        return out

    r, n = int(header["r"]), int(header["n"])
    dec = layers(header["decoder"])
    enc = layers(header["encoder"])
    model = SubspaceModel(r, n, dec, blob(n), blob(n))
    model.encoder = enc
    model.validate()
    if enc:  # SubspaceModel::validate (net.cpp:75-83): encoder chains n -> r
        width = n
        for l in enc:
            if l.W.shape[1] != width or l.b.shape[0] != l.W.shape[0]:
                raise ValueError("model: encoder layer shapes do not chain")
            width = l.W.shape[0]
        if width != r:
            raise ValueError("model: encoder output width != r")
    return model
