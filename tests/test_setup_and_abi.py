"""Host-side checks that need no GPU: the C-ABI library loads and exports every
symbol include/lipsub_b200.h declares; the product's setup (mesh generator,
Xavier decoder, materials, RNG) equals the oracle's; error behaviour mirrors the
reference (ValueError <-> std::invalid_argument)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "lipsub_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lsb_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol(product):
    from paper_2409_03807_b200 import _capi
    lib = ctypes.CDLL(_capi._LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    bound = {name for name, _, _ in _capi.SIGNATURES}
    assert set(syms) == bound, set(syms) ^ bound


def test_oracle_library_is_separate(product):
    """The product library must not contain the oracle."""
    from paper_2409_03807_b200 import _capi
    lib = ctypes.CDLL(_capi._LIB_PATH)
    assert not hasattr(lib, "orc_decode")


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_product_setup_equals_oracle(name, oracle, product):
    from paper_2409_03807_b200 import configs
    pr = configs.build(name)
    ob = oracle.problem(name)
    X, T, Dm, vol, fi = ob.mesh_arrays()
    assert np.array_equal(X, pr.mesh.vertices)
    assert np.array_equal(T, pr.mesh.elements)
    assert np.array_equal(np.nonzero(fi < 0)[0], pr.mesh.pinned)
    layers, shift, scale = ob.decoder_layers()
    assert len(layers) == len(pr.model.decoder)
    for (W, b, act), L in zip(layers, pr.model.decoder):
        assert np.array_equal(W, L.W) and np.array_equal(b, L.b) and act == int(L.act)
    assert np.array_equal(shift, pr.model.norm_shift) and np.array_equal(scale, pr.model.norm_scale)


def test_config_sizes(product):
    """SURVEY §8(a) sizes: c1 (425, 1536, 1020), c2 (18785, 98304, 53040)."""
    from paper_2409_03807_b200 import configs
    for name, (V, E, n, pins) in {"c1": (425, 1536, 1020, 85), "c2": (18785, 98304, 53040, 1105)}.items():
        pr = configs.build(name)
        assert pr.mesh.num_vertices() == V and pr.mesh.num_elements() == E
        assert pr.mesh.num_dofs() == n and pr.mesh.pinned.size == pins
        assert all(L.act == 3 for L in pr.model.decoder[:-1]) and int(pr.model.decoder[-1].act) == 0


def test_config3_mesh_valid_and_material(product, oracle):
    """c3: jittered Kuhn bar passes the det Dm > 1e-14 rule; per-tet E in [5e4, 5e5]."""
    from paper_2409_03807_b200 import lame_from_young, make_bar_mesh
    m = make_bar_mesh(32, 32, 128, 0.25, 0.25, 1.0, jitter_frac=0.1, seed=2)
    assert m.num_vertices() == 140481 and m.num_elements() == 786432 and m.num_dofs() == 408672
    X = m.vertices[m.elements]
    det = np.linalg.det(np.stack([X[:, 1] - X[:, 0], X[:, 2] - X[:, 0], X[:, 3] - X[:, 0]], axis=2))
    assert det.min() > 1e-14
    mu, lam = lame_from_young(m.num_elements(), 5e4, 5e5, 0.35, seed=2)
    E = mu * 2 * 1.35
    assert E.min() >= 5e4 and E.max() <= 5e5
    u = oracle._randu_seq(2, 2, 8)
    assert np.allclose(E[:8], 5e4 + 4.5e5 * u, rtol=1e-15)


def test_gaussian_stream_matches_reference_rng(product, oracle):
    from paper_2409_03807_b200 import configs
    assert np.array_equal(configs.gaussian_latents(3, 4, 5) / 0.5, oracle.randn_seq(3, 0, 20).reshape(4, 5))


def test_solver_config_validation(product):
    """reference SolverConfig::validate (reduced_solver.cpp:14-20)."""
    P = product
    for kw in [dict(epsilon=0.0), dict(max_iters=0), dict(max_linesearch=0), dict(dt=0.0), dict(lbfgs_history=0)]:
        with pytest.raises(ValueError):
            P.SolverConfig(**kw).validate()
    with pytest.raises(ValueError, match="relu"):
        P.lipsub.activation_from_string("relu")


def test_model_validation(product):
    P = product
    mesh = P.make_bar_mesh(2, 1, 1, 1.0, 0.4, 0.3)
    m = P.make_bar_decoder(mesh, 2, 1, 8, P.Activation.Elu, seed=0)
    m.norm_scale[0] = 0.0
    with pytest.raises(ValueError, match="positive"):
        m.validate()


def test_no_cpu_fallback_without_gpu(product):
    """lsb_create must fail loudly when no CUDA device is present (no CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    P = product
    mesh = P.make_bar_mesh(2, 1, 1, 1.0, 0.4, 0.3)
    m = P.make_bar_decoder(mesh, 2, 1, 8, P.Activation.Elu, seed=0)
    with pytest.raises(P.LsbError, match="no CUDA device"):
        P.ReducedSystem(mesh, 1.0, 1.0, 1.0, m)


def test_mesh_errors_mirror_reference(product):
    """build_mesh rejects out-of-range pins (mesh.cpp:136-137)."""
    P = product
    with pytest.raises(RuntimeError, match="pinned vertex"):
        P.build_mesh(np.zeros((4, 3)), np.array([[0, 1, 2, 3]]), [7])
