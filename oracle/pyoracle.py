"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes view of ``oracle/build/liboracle.so``, the plain-C++ restatement of the
reference hps2d hot path (see ``oracle/oracle.hpp`` for the parity status).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs import this module; the product package never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int)


def build() -> None:
    """Compile the oracle with its Makefile (g++ only, seconds)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_last_error.restype = ctypes.c_char_p
        L.oracle_session_create.restype = ctypes.c_void_p
        L.oracle_session_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                            ctypes.c_double, _D, _D, _D, ctypes.c_int]
        for name in ("oracle_session_destroy",):
            getattr(L, name).argtypes = [ctypes.c_void_p]
        L.oracle_dim.restype = ctypes.c_longlong
        L.oracle_dim.argtypes = [ctypes.c_void_p]
        L.oracle_precond_memory.restype = ctypes.c_longlong
        L.oracle_precond_memory.argtypes = [ctypes.c_void_p]
        L.oracle_hierarchy_storage.restype = ctypes.c_longlong
        L.oracle_hierarchy_storage.argtypes = [ctypes.c_void_p]
        L.oracle_set_lean_elements.argtypes = [ctypes.c_int]
        L.oracle_history.restype = ctypes.c_longlong
        L.oracle_history.argtypes = [ctypes.c_void_p, _D, ctypes.c_longlong]
        L.oracle_sample.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_ulonglong, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_double, _D, _D, _D, _I]
        L.oracle_element.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, _D, _D,
                                     _D, _D, _D, _D]
        L.oracle_solve.argtypes = [ctypes.c_void_p, ctypes.c_int, _D, _D, ctypes.c_int,
                                   ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D]
        for name in ("oracle_get_element", "oracle_get_rhs", "oracle_apply_M",
                     "oracle_build_hierarchy", "oracle_level_info", "oracle_level_blocks",
                     "oracle_precond_create", "oracle_precond_apply", "oracle_direct_solve",
                     "oracle_recover", "oracle_dense_M", "oracle_timings",
                     "oracle_level_apply", "oracle_rhs_for_tside"):
            getattr(L, name).argtypes = None  # set per call via explicit casts
        _lib = L
    return _lib


def set_lean_elements(lean: bool) -> None:
    """Keep only T / H per element (no recovery): full-size golden runs."""
    lib().oracle_set_lean_elements(int(lean))


def _p(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(_I)


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().oracle_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)


# ---------------------------------------------------------------- structure
def gll_rule(order: int):
    n = order + 1
    nodes, weights, diff = np.zeros(n), np.zeros(n), np.zeros(n * n)
    _check(lib().oracle_gll_rule(order, _p(nodes), _p(weights), _p(diff)))
    return nodes, weights, diff.reshape(n, n, order="F")


def index_sets(order: int) -> dict:
    m, np1 = order - 1, order + 1
    sizes = [m, m, m, m, m * m, np1 * np1 - 4, np1 * np1]
    out = np.zeros(sum(sizes), dtype=np.int32)
    _check(lib().oracle_index_sets(order, _ip(out)))
    names = ["left", "right", "bottom", "top", "interior", "noncorner", "comp_of_full"]
    res, off = {}, 0
    for name, s in zip(names, sizes):
        res[name] = out[off:off + s].copy()
        off += s
    res["boundary"] = np.concatenate([res["left"], res["right"], res["bottom"], res["top"]])
    return res


def face_graph(n: int) -> dict:
    nf = 2 * n * (n - 1)
    L = 2 * int(np.log2(n))
    faces = np.zeros(6 * nf, dtype=np.int32)
    lr = np.zeros(2 * L, dtype=np.int32)
    foe = np.zeros(4 * n * n, dtype=np.int32)
    _check(lib().oracle_face_graph(n, _ip(faces), _ip(lr), _ip(foe)))
    return {"faces": faces.reshape(nf, 6), "level_range": lr.reshape(L, 2),
            "face_of_element": foe.reshape(n * n, 4)}


# ---------------------------------------------------------------- problems
def sample(kind: int, config: int = 0, seed: int = 0, n: int = 0, order: int = 0,
           kappa: float = 0.0):
    """Seeded samples (coeff real [ne,(N+1)^2], source [ne,(N-1)^2], tside [nrhs,ne,4,N-1])."""
    if kind == 2:
        base_n = [4, 16, 64, 128, 256][config]
        base_o = [8, 16, 16, 20, 12][config]
        n = n or base_n
        order = order or base_o
        nrhs = 32 if config == 4 else 1
    else:
        nrhs = 1
    ne, np1, m = n * n, order + 1, order - 1
    coeff = np.zeros(ne * np1 * np1)
    source = np.zeros(ne * m * m, dtype=np.complex128)
    tside = np.zeros(nrhs * ne * 4 * m, dtype=np.complex128)
    zero = ctypes.c_int(0)
    _check(lib().oracle_sample(kind, config, seed, n, order, kappa, _p(coeff),
                               source.ctypes.data_as(_D), tside.ctypes.data_as(_D),
                               ctypes.byref(zero)))
    return {"n": n, "order": order, "coeff": coeff.reshape(ne, np1 * np1),
            "source": source.reshape(ne, m * m), "tside": tside.reshape(nrhs, ne, 4, m),
            "source_zero": bool(zero.value)}


def element(order: int, h: float, eta: float, coeff_full, interior_src=None):
    """One element's (T, H, pde, I_out) for a complex coefficient on all nodes."""
    np1, m = order + 1, order - 1
    t = np1 * np1 - 4
    c = np.ascontiguousarray(np.broadcast_to(np.asarray(coeff_full, dtype=np.complex128),
                                             (np1 * np1,)))
    src = np.zeros(m * m, dtype=np.complex128) if interior_src is None else \
        np.ascontiguousarray(interior_src, dtype=np.complex128)
    T = np.zeros((4 * m) ** 2, dtype=np.complex128)
    H = np.zeros(4 * m, dtype=np.complex128)
    pde = np.zeros(t * t, dtype=np.complex128)
    iout = np.zeros(4 * m * t, dtype=np.complex128)
    _check(lib().oracle_element(order, h, eta, _p(c.view(np.float64)), _p(src.view(np.float64)),
                                _p(T.view(np.float64)), _p(H.view(np.float64)),
                                _p(pde.view(np.float64)), _p(iout.view(np.float64))))
    return (T.reshape(4 * m, 4 * m, order="F"), H, pde.reshape(t, t, order="F"),
            iout.reshape(4 * m, t, order="F"))


def merge_pair(T1, H1, T2, H2, alpha: int, beta: int, m: int):
    T1 = np.asfortranarray(T1, dtype=np.complex128)
    T2 = np.asfortranarray(T2, dtype=np.complex128)
    H1 = np.ascontiguousarray(H1, dtype=np.complex128)
    H2 = np.ascontiguousarray(H2, dtype=np.complex128)
    T = np.zeros((6 * m, 6 * m), dtype=np.complex128, order="F")
    H = np.zeros(6 * m, dtype=np.complex128)
    _check(lib().oracle_merge_pair(int(m), _p(T1.ravel(order="F").view(np.float64)),
                                   _p(H1.view(np.float64)),
                                   _p(T2.ravel(order="F").view(np.float64)),
                                   _p(H2.view(np.float64)), int(alpha), int(beta),
                                   T.ctypes.data_as(_D), _p(H.view(np.float64))))
    return T, H


class Session:
    """Oracle problem: elements + skeleton (+ hierarchy, preconditioner)."""

    def __init__(self, n, order, kappa, eta, coeff, source, tside, threads: int = 0):
        threads = threads or os.cpu_count() or 1
        self.n, self.order, self.kappa, self.eta = n, order, kappa, eta
        self.m = order - 1
        c = np.ascontiguousarray(coeff, dtype=np.float64).ravel()
        s = np.ascontiguousarray(source, dtype=np.complex128).ravel()
        t = np.ascontiguousarray(tside, dtype=np.complex128).ravel()
        L = lib()
        self._h = L.oracle_session_create(n, order, kappa, eta, _p(c), _p(s.view(np.float64)),
                                          _p(t.view(np.float64)), threads)
        if not self._h:
            raise RuntimeError(L.oracle_last_error().decode())
        self.dim = int(L.oracle_dim(self._h))
        self.nb = 4 * self.m

    @classmethod
    def from_sample(cls, smp: dict, kappa: float, threads: int = 0, rhs_index: int = 0):
        return cls(smp["n"], smp["order"], kappa, kappa, smp["coeff"], smp["source"],
                   smp["tside"][rhs_index], threads)

    def close(self):
        if getattr(self, "_h", None):
            lib().oracle_session_destroy(ctypes.c_void_p(self._h))
            self._h = None

    def __del__(self):
        self.close()

    @property
    def h(self):
        return ctypes.c_void_p(self._h)

    def element(self, e: int):
        T = np.zeros(self.nb * self.nb, dtype=np.complex128)
        H = np.zeros(self.nb, dtype=np.complex128)
        _check(lib().oracle_get_element(self.h, int(e), _p(T.view(np.float64)), _p(H.view(np.float64))))
        return T.reshape(self.nb, self.nb, order="F"), H

    def rhs(self):
        r = np.zeros(self.dim, dtype=np.complex128)
        _check(lib().oracle_get_rhs(self.h, _p(r.view(np.float64))))
        return r

    def rhs_for(self, tside):
        """Skeleton rhs of another impedance datum tside[n^2, 4, N-1] on the same elements."""
        t = np.ascontiguousarray(tside, dtype=np.complex128).ravel()
        r = np.zeros(self.dim, dtype=np.complex128)
        _check(lib().oracle_rhs_for_tside(self.h, _p(t.view(np.float64)), _p(r.view(np.float64))))
        return r

    def apply_M(self, x):
        x = np.ascontiguousarray(x, dtype=np.complex128)
        y = np.zeros(self.dim, dtype=np.complex128)
        _check(lib().oracle_apply_M(self.h, _p(x.view(np.float64)), _p(y.view(np.float64))))
        return y

    def dense_M(self):
        M = np.zeros(self.dim * self.dim, dtype=np.complex128)
        _check(lib().oracle_dense_M(self.h, _p(M.view(np.float64))))
        return M.reshape(self.dim, self.dim, order="F")

    def build_hierarchy(self, depth: int = 0, factor_coarse: bool = True):
        _check(lib().oracle_build_hierarchy(self.h, ctypes.c_int(depth),
                                            ctypes.c_int(int(factor_coarse))))

    def level_blocks(self, level: int) -> tuple[int, dict]:
        nst, first, nf = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(lib().oracle_level_info(self.h, ctypes.c_int(level), ctypes.byref(nst),
                                       ctypes.byref(first), ctypes.byref(nf)))
        bs = 2 * self.m
        keys = np.zeros(2 * nst.value, dtype=np.int32)
        data = np.zeros(nst.value * bs * bs, dtype=np.complex128)
        _check(lib().oracle_level_blocks(self.h, ctypes.c_int(level), _ip(keys),
                                         _p(data.view(np.float64))))
        blocks = {}
        for k in range(nst.value):
            blocks[(int(keys[2 * k]), int(keys[2 * k + 1]))] = \
                data[k * bs * bs:(k + 1) * bs * bs].reshape(bs, bs, order="F")
        return first.value, blocks

    def level_apply(self, level: int, x) -> np.ndarray:
        """y = M_l x on level l's system (faces [first_face, total))."""
        x = np.ascontiguousarray(x, dtype=np.complex128)
        y = np.zeros_like(x)
        _check(lib().oracle_level_apply(self.h, ctypes.c_int(level), _p(x.view(np.float64)),
                                        _p(y.view(np.float64))))
        return y

    def level_dim(self, level: int) -> int:
        nst, first, nf = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(lib().oracle_level_info(self.h, ctypes.c_int(level), ctypes.byref(nst),
                                       ctypes.byref(first), ctypes.byref(nf)))
        return nf.value * 2 * self.m

    def precond(self, depth: int, gamma: int = 1, coarse_iters: int = 4, exact: bool = False):
        _check(lib().oracle_precond_create(self.h, ctypes.c_int(depth), ctypes.c_int(gamma),
                                           ctypes.c_int(coarse_iters), ctypes.c_int(int(exact))))

    def precond_apply(self, v):
        v = np.ascontiguousarray(v, dtype=np.complex128)
        z = np.zeros(self.dim, dtype=np.complex128)
        _check(lib().oracle_precond_apply(self.h, _p(v.view(np.float64)), _p(z.view(np.float64))))
        return z

    def precond_memory(self) -> int:
        return int(lib().oracle_precond_memory(self.h))

    def hierarchy_storage(self) -> int:
        return int(lib().oracle_hierarchy_storage(self.h))

    def solve(self, rhs, preconditioned=True, restart: int = 60, tol: float = 1e-8,
              max_iters: int = 2000, reorth: bool = True, record_history: bool = False):
        """preconditioned: False/0 gmres, True/1 fgmres (flexible, the session
        preconditioner), 2 or "right": gmres with the preconditioner on the right."""
        mode = 2 if preconditioned == "right" else int(preconditioned)
        rhs = np.ascontiguousarray(rhs, dtype=np.complex128)
        x = np.zeros(self.dim, dtype=np.complex128)
        stats = np.zeros(5)
        _check(lib().oracle_solve(self.h, mode, _p(rhs.view(np.float64)),
                                  _p(x.view(np.float64)), restart, tol, max_iters, int(reorth),
                                  int(record_history), _p(stats)))
        rep = {"iterations": int(stats[0]), "converged": bool(stats[1]),
               "final_residual": float(stats[2]), "seconds": float(stats[3]),
               "basis_orthogonality": float(stats[4])}
        if record_history:
            n = int(lib().oracle_history(self.h, None, 0))
            hist = np.zeros(n)
            if n:
                lib().oracle_history(self.h, _p(hist), n)
            rep["residual_history"] = hist.tolist()
        return x, rep

    def direct_solve(self, rhs):
        rhs = np.ascontiguousarray(rhs, dtype=np.complex128)
        x = np.zeros(self.dim, dtype=np.complex128)
        _check(lib().oracle_direct_solve(self.h, _p(rhs.view(np.float64)), _p(x.view(np.float64))))
        return x

    def recover(self, g):
        g = np.ascontiguousarray(g, dtype=np.complex128)
        t = (self.order + 1) ** 2 - 4
        f = np.zeros(self.n * self.n * t, dtype=np.complex128)
        _check(lib().oracle_recover(self.h, _p(g.view(np.float64)), _p(f.view(np.float64))))
        return f.reshape(self.n * self.n, t)

    def timings(self):
        t = np.zeros(3)
        lib().oracle_timings(self.h, _p(t))
        return {"elements": t[0], "skeleton": t[1], "hierarchy": t[2]}
