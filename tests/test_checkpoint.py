"""LIPSUBCKPT1 checkpoints (reference net.cpp:259-353): byte layout, round trip, error types.
CPU only; the GPU test runs the solver from a loaded checkpoint."""
import json
import struct

import numpy as np
import pytest

import paper_2409_03807_b200 as P
from conftest import rel_err


def _tiny_model(r=3, n=7, width=5, seed=2):
    rng = np.random.default_rng(seed)
    dims = [r, width, width, n]
    acts = [P.Activation.Silu, P.Activation.Tanh, P.Activation.Identity]
    layers = [P.Layer(rng.standard_normal((dims[i + 1], dims[i])), rng.standard_normal(dims[i + 1]), acts[i])
              for i in range(3)]
    return P.SubspaceModel(r, n, layers, rng.standard_normal(n), 0.5 + rng.random(n))


def _write_by_hand(path, m, encoder=()):
    """Independent byte-level writer of the reference layout (not the module's writer)."""
    names = {0: "identity", 1: "silu", 2: "tanh", 3: "elu"}
    meta = lambda ls: [{"rows": l.W.shape[0], "cols": l.W.shape[1], "act": names[int(l.act)]} for l in ls]
    hs = json.dumps({"format": "lipsub-checkpoint", "r": m.r, "n": m.n, "decoder": meta(m.decoder),
                     "encoder": meta(encoder)}).encode()
    with open(path, "wb") as f:
        f.write(b"LIPSUBCKPT1\n" + struct.pack("<Q", len(hs)) + hs)
        for l in list(m.decoder) + list(encoder):
            for i in range(l.W.shape[0]):
                for j in range(l.W.shape[1]):
                    f.write(struct.pack("<d", l.W[i, j]))
            for v in l.b:
                f.write(struct.pack("<d", v))
        for v in list(m.norm_shift) + list(m.norm_scale):
            f.write(struct.pack("<d", v))


def _same(a, b):
    assert a.r == b.r and a.n == b.n and len(a.decoder) == len(b.decoder)
    for la, lb in zip(a.decoder, b.decoder):
        assert np.array_equal(la.W, lb.W) and np.array_equal(la.b, lb.b) and int(la.act) == int(lb.act)
    assert np.array_equal(a.norm_shift, b.norm_shift) and np.array_equal(a.norm_scale, b.norm_scale)


def test_load_reference_layout_bit_exact(tmp_path):
    m = _tiny_model()
    enc = [P.Layer(np.ones((4, 7)), np.zeros(4), P.Activation.Tanh),
           P.Layer(np.ones((3, 4)), np.zeros(3), P.Activation.Identity)]
    p = tmp_path / "model.ckpt"
    _write_by_hand(p, m, enc)
    got = P.load_checkpoint(str(p))
    _same(got, m)
    assert len(got.encoder) == 2 and got.encoder[0].W.shape == (4, 7)


def test_round_trip_and_writer_matches_reference_bytes(tmp_path):
    m = _tiny_model(seed=5)
    a, b = tmp_path / "a.ckpt", tmp_path / "b.ckpt"
    P.save_checkpoint(m, str(a))
    _same(P.load_checkpoint(str(a)), m)
    _write_by_hand(b, m)
    # identical blobs (headers may differ only in JSON whitespace)
    da, db = a.read_bytes(), b.read_bytes()
    ha, hb = struct.unpack_from("<Q", da, 12)[0], struct.unpack_from("<Q", db, 12)[0]
    assert json.loads(da[20:20 + ha]) == json.loads(db[20:20 + hb])
    assert da[20 + ha:] == db[20 + hb:]


def test_checkpoint_errors(tmp_path):
    m = _tiny_model()
    p = tmp_path / "m.ckpt"
    P.save_checkpoint(m, str(p))
    raw = p.read_bytes()
    (tmp_path / "magic.ckpt").write_bytes(b"NOTCKPT....\n" + raw[12:])
    with pytest.raises(RuntimeError, match="bad magic"):
        P.load_checkpoint(str(tmp_path / "magic.ckpt"))
    (tmp_path / "trunc.ckpt").write_bytes(raw[:-8])
    with pytest.raises(RuntimeError, match="truncated"):
        P.load_checkpoint(str(tmp_path / "trunc.ckpt"))
    with pytest.raises(RuntimeError, match="cannot open"):
        P.load_checkpoint(str(tmp_path / "missing.ckpt"))
    bad = raw.replace(b'"silu"', b'"relu"')
    (tmp_path / "relu.ckpt").write_bytes(bad)
    with pytest.raises(ValueError, match="relu"):
        P.load_checkpoint(str(tmp_path / "relu.ckpt"))
    m.norm_scale[0] = -1.0
    with pytest.raises(ValueError):
        P.save_checkpoint(m, str(tmp_path / "neg.ckpt"))


@pytest.mark.gpu
def test_solver_from_checkpoint_matches_in_memory_model(tmp_path, product):
    """A config-2 decoder written and reloaded drives the device objective bit-identically."""
    from paper_2409_03807_b200 import configs
    pr = configs.build("c1")
    p = tmp_path / "c1.ckpt"
    P.save_checkpoint(pr.model, str(p))
    m2 = P.load_checkpoint(str(p))
    s1 = pr.system("fp64")
    s2 = P.ReducedSystem(pr.mesh, pr.mu, pr.lam, pr.spec.density, m2, "fp64")
    z = 0.3 * np.ones(pr.model.r)
    E1, g1 = s1.eval(z)
    E2, g2 = s2.eval(z)
    assert E1 == E2 and np.array_equal(g1, g2)
