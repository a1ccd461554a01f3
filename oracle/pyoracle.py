"""TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.

ctypes wrapper of the CPU oracle (oracle/liblipsub_oracle.so, a C++ restatement
of the reference hot path; see oracle/oracle.hpp for provenance and the parity
pin).  Imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liblipsub_oracle.so")

_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_lib = None

OBJECTIVE_CB = C.CFUNCTYPE(C.c_double, _D, _D, C.c_int, C.c_void_p)
HESSIAN_CB = C.CFUNCTYPE(None, _D, _D, C.c_int, C.c_void_p)


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        sigs = {
            "orc_last_error": (C.c_char_p, []),
            "orc_randn_seq": (None, [C.c_uint64, C.c_uint64, C.c_int, _D]),
            "orc_activation_eval": (C.c_double, [C.c_int, C.c_double, C.c_int]),
            "orc_ctx_bar": (C.c_void_p, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                         C.c_double, C.c_uint64, C.c_int]),
            "orc_ctx_mesh": (C.c_void_p, [C.c_int, _D, C.c_int, _I, C.c_int, _I]),
            "orc_ctx_free": (None, [C.c_void_p]),
            "orc_ctx_info": (None, [C.c_void_p, _I, _I, _I, _I]),
            "orc_ctx_mesh_arrays": (None, [C.c_void_p, _D, _I, _D, _D, _I]),
            "orc_ctx_set_material": (C.c_int, [C.c_void_p, _D, _D, C.c_double]),
            "orc_ctx_mass": (None, [C.c_void_p, _D, _D]),
            "orc_ctx_set_pins": (None, [C.c_void_p, _D]),
            "orc_ctx_set_decoder": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _I, _I, C.POINTER(_D), C.POINTER(_D),
                                              _I, _D, _D]),
            "orc_ctx_bar_decoder": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                              C.c_double]),
            "orc_ctx_decoder_layer": (None, [C.c_void_p, C.c_int, _I, _I, _I, _D, _D]),
            "orc_ctx_decoder_layers": (C.c_int, [C.c_void_p]),
            "orc_ctx_decoder_norm": (None, [C.c_void_p, _D, _D]),
            "orc_element_snh": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_double, _D, C.c_int, _D, _D, _D]),
            "orc_assemble": (C.c_int, [C.c_void_p, _D, C.c_int, _I, _D, _D, _D]),
            "orc_elastic_hessian_apply": (C.c_int, [C.c_void_p, _D, C.c_int, _D, _D]),
            "orc_decode": (C.c_int, [C.c_void_p, _D, _D]),
            "orc_decode_jacobian": (C.c_int, [C.c_void_p, _D, _D]),
            "orc_decode_second_directional": (C.c_int, [C.c_void_p, _D, _D, _D, _D]),
            "orc_objective_eval": (C.c_int, [C.c_void_p, _D, C.c_double, _D, _D, _D]),
            "orc_objective_hessian": (C.c_int, [C.c_void_p, _D, C.c_double, _D, _D]),
            "orc_project_spd": (C.c_int, [_D, C.c_int, _D]),
            "orc_set_cubature": (C.c_int, [C.c_void_p, C.c_int, _I, _D]),
            "orc_projective_newton": (C.c_int, [OBJECTIVE_CB, HESSIAN_CB, C.c_void_p, C.c_int, _D, C.c_double,
                                                C.c_int, C.c_int, _I, _I, _D]),
            "orc_objective_projective_newton": (C.c_int, [C.c_void_p, _D, C.c_double, _D, C.c_double, C.c_int,
                                                          C.c_int, _I, _I, _D, _I, _I]),
            "orc_objective_eval_batch": (C.c_int, [C.c_void_p, _D, C.c_double, C.c_int, _D, _D, _D, C.c_int]),
            "orc_lbfgs_minimize": (C.c_int, [OBJECTIVE_CB, C.c_void_p, C.c_int, _D, C.c_double, C.c_int, C.c_int,
                                             C.c_int, _I, _I, _D]),
            "orc_simulate": (C.c_int, [C.c_void_p, _D, C.c_double, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                       C.c_int, _D, _D, _D, _I, _I, _D, _D, _I, _I, _D]),
            "orc_reduced_potential_hessian": (C.c_int, [C.c_void_p, _D, _D]),
            "orc_lipschitz_loss2": (C.c_int, [C.c_void_p, C.c_int, _D, _D, C.c_int, _D]),
            "orc_elastic_third_contraction": (C.c_int, [C.c_void_p, _D, C.c_int, _D, _D, _D]),
            "orc_lipschitz_loss2_grad": (C.c_int, [C.c_void_p, C.c_int, _D, _D, C.c_int, _D, _D]),
            "orc_reduced_step": (C.c_int, [C.c_void_p, _D, _D, C.c_double, C.c_int, C.c_int, C.c_int, C.c_double,
                                           C.c_int, _D, _D, _D, _I, _I]),
            "orc_hardware_threads": (C.c_int, []),
        }
        for name, (res, args) in sigs.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _chk(rc):
    if rc != 0:
        msg = lib().orc_last_error().decode()
        if "must be" in msg or "wrong length" in msg or "coincident" in msg or "no pairs" in msg \
                or "do not chain" in msg or "order" in msg:
            raise ValueError(msg)
        raise OracleError(msg)


def _d(a):
    return None if a is None else a.ctypes.data_as(_D)


def _i(a):
    return None if a is None else a.ctypes.data_as(_I)


def randn_seq(seed, tag, count):
    out = np.zeros(count)
    lib().orc_randn_seq(seed, tag, count, _d(out))
    return out


def activation_eval(act, x, order):
    return lib().orc_activation_eval(int(act), float(x), int(order))


class Oracle:
    """One problem instance (mesh + material + decoder) in the CPU oracle."""

    def __init__(self, handle):
        if not handle:
            raise OracleError(lib().orc_last_error().decode())
        self.h = handle
        V, E, nf, npin = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        lib().orc_ctx_info(self.h, C.byref(V), C.byref(E), C.byref(nf), C.byref(npin))
        self.V, self.E, self.n_free, self.npinned = V.value, E.value, nf.value, npin.value
        self.n = 3 * self.n_free
        self.r = None

    @classmethod
    def bar(cls, nx, ny, nz, w=0.25, h=0.25, d=1.0, jitter=0.0, seed=0, pin_left=True):
        return cls(lib().orc_ctx_bar(nx, ny, nz, w, h, d, jitter, seed, int(pin_left)))

    @classmethod
    def from_mesh(cls, X, T, pins):
        X = np.ascontiguousarray(X, np.float64)
        T = np.ascontiguousarray(T, np.int32)
        pins = np.ascontiguousarray(pins, np.int32)
        p = pins if pins.size else np.zeros(1, np.int32)
        return cls(lib().orc_ctx_mesh(X.shape[0], _d(X), T.shape[0], _i(T), pins.size, _i(p)))

    def __del__(self):
        try:
            lib().orc_ctx_free(self.h)
        except Exception:
            pass

    def mesh_arrays(self):
        X = np.zeros((self.V, 3))
        T = np.zeros((self.E, 4), np.int32)
        Dm = np.zeros((self.E, 3, 3))
        vol = np.zeros(self.E)
        fi = np.zeros(self.V, np.int32)
        lib().orc_ctx_mesh_arrays(self.h, _d(X), _i(T), _d(Dm), _d(vol), _i(fi))
        return X, T, Dm, vol, fi

    def set_material(self, mu, lam, density):
        mu = np.ascontiguousarray(np.broadcast_to(np.asarray(mu, np.float64), (self.E,)))
        lam = np.ascontiguousarray(np.broadcast_to(np.asarray(lam, np.float64), (self.E,)))
        _chk(lib().orc_ctx_set_material(self.h, _d(mu), _d(lam), float(density)))
        self.mass = np.zeros(self.n)
        tot = C.c_double()
        lib().orc_ctx_mass(self.h, _d(self.mass), C.byref(tot))
        self.total_mass = tot.value

    def set_pins(self, pin_positions):
        p = np.ascontiguousarray(pin_positions, np.float64)
        lib().orc_ctx_set_pins(self.h, _d(p))

    def set_decoder(self, layers, shift, scale, r):
        """layers: list of (W rows x cols, b, act)."""
        L = len(layers)
        Ws = [np.ascontiguousarray(W, np.float64) for W, _, _ in layers]
        bs = [np.ascontiguousarray(b, np.float64) for _, b, _ in layers]
        rows = np.array([W.shape[0] for W in Ws], np.int32)
        cols = np.array([W.shape[1] for W in Ws], np.int32)
        acts = np.array([int(a) for _, _, a in layers], np.int32)
        wp = (_D * L)(*[_d(w) for w in Ws])
        bp = (_D * L)(*[_d(b) for b in bs])
        shift = np.ascontiguousarray(shift, np.float64)
        scale = np.ascontiguousarray(scale, np.float64)
        _chk(lib().orc_ctx_set_decoder(self.h, r, L, _i(rows), _i(cols), wp, bp, _i(acts), _d(shift), _d(scale)))
        self.r = r

    def bar_decoder(self, r, hidden, width, act, seed, out_scale=1e-2):
        _chk(lib().orc_ctx_bar_decoder(self.h, r, hidden, width, int(act), seed, out_scale))
        self.r = r

    def decoder_layers(self):
        out = []
        for l in range(lib().orc_ctx_decoder_layers(self.h)):
            rows, cols, act = C.c_int(), C.c_int(), C.c_int()
            lib().orc_ctx_decoder_layer(self.h, l, C.byref(rows), C.byref(cols), C.byref(act), None, None)
            W = np.zeros((rows.value, cols.value))
            b = np.zeros(rows.value)
            lib().orc_ctx_decoder_layer(self.h, l, C.byref(rows), C.byref(cols), C.byref(act), _d(W), _d(b))
            out.append((W, b, act.value))
        shift = np.zeros(self.n)
        scale = np.zeros(self.n)
        lib().orc_ctx_decoder_norm(self.h, _d(shift), _d(scale))
        return out, shift, scale

    # ---- primitives
    def element_snh(self, e, mu, lam, positions, want_hess=True):
        pos = np.ascontiguousarray(positions, np.float64)
        en = C.c_double()
        g = np.zeros(12)
        H = np.zeros((12, 12))
        _chk(lib().orc_element_snh(self.h, e, mu, lam, _d(pos), int(want_hess), C.byref(en), _d(g), _d(H)))
        return en.value, g, H

    def assemble(self, q, subset=None, weights=None):
        q = np.ascontiguousarray(q, np.float64)
        v = C.c_double()
        g = np.zeros(self.n)
        if subset is None:
            _chk(lib().orc_assemble(self.h, _d(q), -1, None, None, C.byref(v), _d(g)))
        else:
            ids = np.ascontiguousarray(subset, np.int32)
            w = np.ascontiguousarray(weights, np.float64)
            _chk(lib().orc_assemble(self.h, _d(q), ids.size, _i(ids) if ids.size else None,
                                    _d(w) if ids.size else None, C.byref(v), _d(g)))
        return v.value, g

    def hessian_apply(self, q, Y):
        q = np.ascontiguousarray(q, np.float64)
        Y = np.ascontiguousarray(Y, np.float64)
        out = np.zeros_like(Y)
        _chk(lib().orc_elastic_hessian_apply(self.h, _d(q), Y.shape[1], _d(Y), _d(out)))
        return out

    def decode(self, z):
        q = np.zeros(self.n)
        _chk(lib().orc_decode(self.h, _d(np.ascontiguousarray(z, np.float64)), _d(q)))
        return q

    def decode_jacobian(self, z):
        J = np.zeros((self.n, self.r))
        _chk(lib().orc_decode_jacobian(self.h, _d(np.ascontiguousarray(z, np.float64)), _d(J)))
        return J

    def decode_second_directional(self, z, u, v):
        out = np.zeros(self.n)
        _chk(lib().orc_decode_second_directional(self.h, _d(np.ascontiguousarray(z, np.float64)),
                                                 _d(np.ascontiguousarray(u, np.float64)),
                                                 _d(np.ascontiguousarray(v, np.float64)), _d(out)))
        return out

    def eval(self, z, qbar=None, dt=0.05, want_grad=True):
        v = C.c_double()
        g = np.zeros(self.r) if want_grad else None
        qb = None if qbar is None else np.ascontiguousarray(qbar, np.float64)
        _chk(lib().orc_objective_eval(self.h, _d(qb), dt, _d(np.ascontiguousarray(z, np.float64)), C.byref(v),
                                      _d(g)))
        return (v.value, g) if want_grad else v.value

    def hessian(self, z, qbar=None, dt=0.05):
        H = np.zeros((self.r, self.r))
        qb = None if qbar is None else np.ascontiguousarray(qbar, np.float64)
        _chk(lib().orc_objective_hessian(self.h, _d(qb), dt, _d(np.ascontiguousarray(z, np.float64)), _d(H)))
        return H

    def set_cubature(self, ids=None, weights=None):
        if ids is None:
            _chk(lib().orc_set_cubature(self.h, 0, None, None))
            return
        ids = np.ascontiguousarray(ids, np.int32)
        w = np.ascontiguousarray(weights, np.float64)
        _chk(lib().orc_set_cubature(self.h, int(ids.size), ids.ctypes.data_as(_I), _d(w)))

    def projective_newton(self, z0, qbar=None, dt=0.05, epsilon=1e-5, max_iters=1024, max_ls=128):
        """projective_newton_minimize on this problem's ReducedObjective (reduced_solver.cpp:133-182)."""
        z = np.ascontiguousarray(z0, np.float64).copy()
        qb = None if qbar is None else np.ascontiguousarray(qbar, np.float64)
        code, it, gn, ev, vev = C.c_int(), C.c_int(), C.c_double(), C.c_int(), C.c_int()
        _chk(lib().orc_objective_projective_newton(self.h, _d(qb), dt, _d(z), epsilon, max_iters, max_ls,
                                                   C.byref(code), C.byref(it), C.byref(gn), C.byref(ev),
                                                   C.byref(vev)))
        return {"z": z, "code": code.value, "iterations": it.value, "gnorm": gn.value, "evals": ev.value,
                "value_evals": vev.value}

    def eval_batch(self, Z, qbar=None, dt=0.05, want_grad=True, threads=1):
        Z = np.ascontiguousarray(Z, np.float64)
        B = Z.shape[0]
        E = np.zeros(B)
        G = np.zeros((B, self.r)) if want_grad else None
        qb = None if qbar is None else np.ascontiguousarray(qbar, np.float64)
        _chk(lib().orc_objective_eval_batch(self.h, _d(qb), dt, B, _d(Z), _d(E), _d(G), threads))
        return (E, G) if want_grad else E

    def simulate(self, steps, cfg, gravity=(0, 0, -9.8), positions=None, velocities=None, z=None,
                 quasi_static=False):
        pos = np.ascontiguousarray(positions if positions is not None else self.mesh_arrays()[0], np.float64).copy()
        vel = np.ascontiguousarray(velocities if velocities is not None else np.zeros((self.V, 3)), np.float64).copy()
        zz = np.ascontiguousarray(z if z is not None else np.zeros(self.r), np.float64).copy()
        codes = np.zeros(steps, np.int32)
        iters = np.zeros(steps, np.int32)
        gn = np.zeros(steps)
        ms = np.zeros(steps)
        ev = np.zeros(steps, np.int32)
        vev = np.zeros(steps, np.int32)
        zt = np.zeros((steps, self.r))
        g = np.ascontiguousarray(gravity, np.float64)
        _chk(lib().orc_simulate(self.h, _d(g), cfg.epsilon, cfg.max_iters, cfg.max_linesearch, cfg.lbfgs_history,
                                cfg.dt, int(quasi_static), steps, _d(pos), _d(vel), _d(zz), _i(codes), _i(iters),
                                _d(gn), _d(ms), _i(ev), _i(vev), _d(zt)))
        return dict(positions=pos, velocities=vel, z=zz, codes=codes, iterations=iters, gnorm=gn, wall_ms=ms,
                    grad_evals=ev, value_evals=vev, z_traj=zt)

    def reduced_step(self, positions, velocities, z, pin_positions, force, cfg, quasi_static=False):
        """One reduced_step with an explicit frame; returns (positions, velocities, z, code, iters)."""
        pos = np.ascontiguousarray(positions, np.float64).copy()
        vel = np.ascontiguousarray(velocities, np.float64).copy()
        zz = np.ascontiguousarray(z, np.float64).copy()
        pins = np.ascontiguousarray(pin_positions, np.float64)
        f = np.ascontiguousarray(force, np.float64)
        code, iters = C.c_int(), C.c_int()
        _chk(lib().orc_reduced_step(self.h, _d(pins), _d(f), cfg.epsilon, cfg.max_iters, cfg.max_linesearch,
                                    cfg.lbfgs_history, cfg.dt, int(quasi_static), _d(pos), _d(vel), _d(zz),
                                    C.byref(code), C.byref(iters)))
        return pos, vel, zz, code.value, iters.value

    def reduced_potential_hessian(self, z):
        H = np.zeros((self.r, self.r))
        _chk(lib().orc_reduced_potential_hessian(self.h, _d(np.ascontiguousarray(z, np.float64)), _d(H)))
        return H

    def lipschitz_loss2(self, Z1, Z2, threads=1):
        Z1 = np.ascontiguousarray(Z1, np.float64)
        Z2 = np.ascontiguousarray(Z2, np.float64)
        out = C.c_double()
        _chk(lib().orc_lipschitz_loss2(self.h, Z1.shape[0], _d(Z1), _d(Z2), threads, C.byref(out)))
        return out.value

    def third_contraction(self, q, A, B):
        """elastic_third_contraction (energy.cpp:495-510) at configuration q."""
        q = np.ascontiguousarray(q, np.float64)
        A = np.ascontiguousarray(A, np.float64)
        B = np.ascontiguousarray(B, np.float64)
        out = np.zeros(self.n)
        _chk(lib().orc_elastic_third_contraction(self.h, _d(q), A.shape[1], _d(A), _d(B), _d(out)))
        return out

    def lipschitz_loss2_grad(self, Z1, Z2, threads=1):
        """(loss, [(dW, db) per decoder layer]) of the order-2 Lipschitz loss."""
        Z1 = np.ascontiguousarray(Z1, np.float64)
        Z2 = np.ascontiguousarray(Z2, np.float64)
        layers = self.decoder_layers()[0]
        flat = np.zeros(sum(W.size + b.size for W, b, _ in layers))
        out = C.c_double()
        _chk(lib().orc_lipschitz_loss2_grad(self.h, Z1.shape[0], _d(Z1), _d(Z2), threads, C.byref(out), _d(flat)))
        grads, o = [], 0
        for W, b, _ in layers:
            gW = flat[o:o + W.size].reshape(W.shape)
            o += W.size
            grads.append((gW, flat[o:o + b.size].copy()))
            o += b.size
        return out.value, grads


def project_spd(H):
    """project_spd (energy.cpp:370-380)."""
    H = np.ascontiguousarray(H, np.float64)
    out = np.zeros_like(H)
    _chk(lib().orc_project_spd(_d(H), H.shape[0], _d(out)))
    return out


def projective_newton_minimize(fn, hess, x, epsilon=1e-5, max_iters=1024, max_ls=128):
    """Oracle projective Newton on Python callbacks fn(x, grad_or_None) and hess(x) -> H."""
    n = x.shape[0]

    def cb(xp, gp, nn, user):
        xv = np.ctypeslib.as_array(xp, shape=(nn,)).copy()
        if gp:
            g = np.zeros(nn)
            v = fn(xv, g)
            np.ctypeslib.as_array(gp, shape=(nn,))[:] = g
            return v
        return fn(xv, None)

    def hcb(xp, hp, nn, user):
        xv = np.ctypeslib.as_array(xp, shape=(nn,)).copy()
        np.ctypeslib.as_array(hp, shape=(nn * nn,))[:] = np.asarray(hess(xv), np.float64).reshape(-1)

    cbf, hcf = OBJECTIVE_CB(cb), HESSIAN_CB(hcb)
    xx = np.ascontiguousarray(x, np.float64).copy()
    code, it, gn = C.c_int(), C.c_int(), C.c_double()
    _chk(lib().orc_projective_newton(cbf, hcf, None, n, _d(xx), epsilon, max_iters, max_ls, C.byref(code),
                                     C.byref(it), C.byref(gn)))
    return xx, {"code": code.value, "iterations": it.value, "gnorm": gn.value}


def lbfgs_minimize(fn, x, epsilon=1e-5, max_iters=1024, max_ls=128, history=8):
    """Oracle L-BFGS on a Python objective fn(x, grad_or_None) -> value."""
    n = x.shape[0]

    def cb(xp, gp, nn, user):
        xv = np.ctypeslib.as_array(xp, shape=(nn,)).copy()
        if gp:
            g = np.zeros(nn)
            v = fn(xv, g)
            np.ctypeslib.as_array(gp, shape=(nn,))[:] = g
            return v
        return fn(xv, None)

    cbf = OBJECTIVE_CB(cb)
    xx = np.ascontiguousarray(x, np.float64).copy()
    code, it, gn = C.c_int(), C.c_int(), C.c_double()
    _chk(lib().orc_lbfgs_minimize(cbf, None, n, _d(xx), epsilon, max_iters, max_ls, history, C.byref(code),
                                  C.byref(it), C.byref(gn)))
    return xx, code.value, it.value, gn.value


def problem(name):
    """The BASELINE.json config as an oracle instance (mirrors paper_2409_03807_b200.configs)."""
    specs = {
        "c1": ((4, 4, 16), 8, 5, 64, 0, 0.0, (1e5, 1e5)),
        "c2": ((16, 16, 64), 16, 5, 128, 1, 0.0, (1e5, 1e5)),
        "c3": ((32, 32, 128), 32, 5, 256, 2, 0.1, (5e4, 5e5)),
    }
    (nx, ny, nz), r, hid, width, seed, jit, (elo, ehi) = specs[name]
    o = Oracle.bar(nx, ny, nz, 0.25, 0.25, 1.0, jit, seed, True)
    nu = 0.35
    if ehi > elo:
        u = _randu_seq(seed, 2, o.E)
        E = elo + (ehi - elo) * u
    else:
        E = np.full(o.E, elo)
    mu = E / (2 * (1 + nu))
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    o.set_material(mu, lam, 1000.0)
    o.bar_decoder(r, hid, width, 3, seed, 1e-2)
    return o


def _randu_seq(seed, tag, count):
    out = np.zeros(count)
    L = lib()
    fn = L.orc_randu_seq
    fn.restype = C.c_double
    fn.argtypes = [C.c_uint64, C.c_uint64, C.c_int, _D]
    fn(seed, tag, count, _d(out))
    return out
