"""hps_b200 — B200-native HPS-multigrid hot path (arXiv 2511.00735).

Python mirror of the reference hps2d C++ entry points on the hot path, bound
through the C ABI in ``include/hps_b200.h`` (``libhps_b200.so``, built for
sm_100a by ``make -C paper_2511_00735_b200``).  Names follow the reference:

    build_elements      ElementOperators / build_elements   proj/src/element.cpp:127-174, mesh.cpp:36-109
    assemble_skeleton   SkeletonSystem + BlockMatrix::apply proj/src/skeleton.cpp:88-137, block_matrix.cpp:23-31
    build_hierarchy     build_hierarchy / eliminate_level   proj/src/dissection.cpp:153-227
    merge_pair          merge_pair                          proj/src/dissection.cpp:23-82
    build_preconditioner MgPreconditioner                   proj/src/multigrid.cpp:9-100
    fgmres / gmres      gmres_driver                        proj/src/krylov.cpp:45-192

There is no CPU fallback: every call goes to the CUDA library, and importing
this module fails loudly when the library has not been built.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhps_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"hps_b200: {LIB_PATH} is missing; build it with "
                      f"`make -C {_HERE}` (nvcc, sm_100a) or __graft_entry__.build()")

_lib = ctypes.CDLL(LIB_PATH)
_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int)
_VP = ctypes.c_void_p

OK, INVALID_ARGUMENT, NO_CONVERGENCE, IO_ERROR, INTERNAL = range(5)


class HpsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class MgConfig(ctypes.Structure):
    """MgConfig (proj/include/hps/multigrid.hpp:12-18)."""
    _fields_ = [("depth", ctypes.c_int), ("gamma", ctypes.c_int),
                ("coarse_iters", ctypes.c_int), ("exact_coarse", ctypes.c_int)]


class KrylovConfig(ctypes.Structure):
    """KrylovConfig (proj/include/hps/krylov.hpp:15-21)."""
    _fields_ = [("restart", ctypes.c_int), ("tol", ctypes.c_double), ("max_iters", ctypes.c_int),
                ("record_history", ctypes.c_int), ("reorthogonalize", ctypes.c_int)]


class SolveReport(ctypes.Structure):
    """SolveReport (proj/include/hps/krylov.hpp:23-34), device-timed."""
    _fields_ = [("iterations", ctypes.c_int), ("converged", ctypes.c_int),
                ("final_residual", ctypes.c_double), ("seconds", ctypes.c_double),
                ("precond_seconds", ctypes.c_double), ("matvec_seconds", ctypes.c_double),
                ("wall_build", ctypes.c_double), ("wall_solve", ctypes.c_double),
                ("precond_memory", ctypes.c_int64), ("basis_orthogonality", ctypes.c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


def _sig(name, restype, *argtypes):
    f = getattr(_lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


_st = ctypes.c_int
_sig("hpsb_last_error", ctypes.c_char_p)
_sig("hpsb_version", ctypes.c_char_p)
_sig("hpsb_context_create", _st, ctypes.c_int, ctypes.POINTER(_VP))
_sig("hpsb_context_destroy", _st, _VP)
_sig("hpsb_context_synchronize", _st, _VP)
_sig("hpsb_context_launches", ctypes.c_int64, _VP)
_sig("hpsb_context_residual_history", ctypes.c_int64, _VP, _D, ctypes.c_int64)
_sig("hpsb_gll_rule", _st, ctypes.c_int, _D, _D, _D)
_sig("hpsb_index_sets", _st, ctypes.c_int, _I)
_sig("hpsb_face_graph", _st, ctypes.c_int, _I, _I, _I)
_sig("hpsb_problem_dims", _st, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _I, _I, _I,
     _D, _I, _D)
_sig("hpsb_problem_sample", _st, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
     ctypes.c_int, ctypes.c_double, _D, _D, _D, _I)
_sig("hpsb_elements_build", _st, _VP, ctypes.c_int, ctypes.c_int, ctypes.c_double, _D, _D,
     ctypes.POINTER(_VP))
_sig("hpsb_elements_build_dev", _st, _VP, ctypes.c_int, ctypes.c_int, ctypes.c_double, _VP, _VP,
     ctypes.POINTER(_VP))
_sig("hpsb_elements_destroy", _st, _VP)
_sig("hpsb_elements_get", _st, _VP, ctypes.c_int, ctypes.c_int, _D, _D)
_sig("hpsb_skeleton_create", _st, _VP, _D, ctypes.c_int, ctypes.POINTER(_VP))
_sig("hpsb_elements_fallbacks", _st, _VP, ctypes.POINTER(ctypes.c_int))
_sig("hpsb_skeleton_create_boundary", _st, _VP, _D, ctypes.c_int, ctypes.POINTER(_VP))
_sig("hpsb_skeleton_destroy", _st, _VP)
_sig("hpsb_skeleton_dim", ctypes.c_int64, _VP)
_sig("hpsb_skeleton_rhs", _st, _VP, ctypes.c_int, _D)
_sig("hpsb_skeleton_rhs_dev", _VP, _VP, ctypes.c_int)
_sig("hpsb_skeleton_apply", _st, _VP, _D, _D)
_sig("hpsb_skeleton_apply_dev", _st, _VP, _VP, _VP)
_sig("hpsb_recover", _st, _VP, _D, ctypes.c_int, _D)
_sig("hpsb_recover_dev", _st, _VP, _VP, ctypes.c_int, _VP)
_sig("hpsb_hierarchy_build", _st, _VP, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_VP))
_sig("hpsb_hierarchy_destroy", _st, _VP)
_sig("hpsb_hierarchy_info", _st, _VP, _I, _I, ctypes.POINTER(ctypes.c_int64), _D)
_sig("hpsb_hierarchy_level_blocks", _st, _VP, ctypes.c_int, _I, _I, _I, _D)
_sig("hpsb_hierarchy_level_apply", _st, _VP, ctypes.c_int, _D, _D)
_sig("hpsb_merge_pair", _st, _VP, ctypes.c_int, _D, _D, _D, _D, ctypes.c_int, ctypes.c_int, _D, _D)
_sig("hpsb_precond_create", _st, _VP, MgConfig, ctypes.POINTER(_VP))
_sig("hpsb_precond_destroy", _st, _VP)
_sig("hpsb_precond_apply", _st, _VP, _D, _D)
_sig("hpsb_direct_solve", _st, _VP, _D, _D)
_sig("hpsb_skeleton_apply_batch_dev", _st, _VP, _VP, _VP, ctypes.c_int)
_sig("hpsb_precond_apply_batch_dev", _st, _VP, _VP, _VP, ctypes.c_int)
_sig("hpsb_direct_solve_dev", _st, _VP, _VP, _VP)
_sig("hpsb_precond_apply_dev", _st, _VP, _VP, _VP)
_sig("hpsb_fgmres", _st, _VP, _VP, _D, _D, KrylovConfig, ctypes.POINTER(SolveReport))
_sig("hpsb_fgmres_dev", _st, _VP, _VP, _VP, _VP, KrylovConfig, ctypes.POINTER(SolveReport))
_sig("hpsb_gmres", _st, _VP, _VP, _D, _D, KrylovConfig, ctypes.POINTER(SolveReport))
_sig("hpsb_gmres_dev", _st, _VP, _VP, _VP, _VP, KrylovConfig, ctypes.POINTER(SolveReport))
_sig("hpsb_fgmres_batch", _st, _VP, _VP, _D, _D, ctypes.c_int, KrylovConfig,
     ctypes.POINTER(SolveReport))
_sig("hpsb_fgmres_batch_dev", _st, _VP, _VP, _VP, _VP, ctypes.c_int, KrylovConfig,
     ctypes.POINTER(SolveReport))
_sig("hpsb_context_timer_start", _st, _VP)
_sig("hpsb_context_timer_stop", _st, _VP, _D)
_sig("hpsb_context_profile", _st, _VP, ctypes.c_int)
_sig("hpsb_context_profile_count", ctypes.c_int, _VP)
_sig("hpsb_context_profile_entry", _st, _VP, ctypes.c_int, ctypes.c_char_p, ctypes.c_int,
     ctypes.POINTER(ctypes.c_int64), _D, _D, _D)
_sig("hpsb_context_profile_reset", _st, _VP)
_sig("hpsb_precond_bytes", ctypes.c_int64, _VP)
_sig("hpsb_nccl_unique_id", _st, ctypes.c_char_p)
_sig("hpsb_context_attach_nccl", _st, _VP, ctypes.c_char_p, ctypes.c_int, ctypes.c_int)
_sig("hpsb_local_group_create", _st, ctypes.c_int, ctypes.POINTER(_VP))
_sig("hpsb_local_group_destroy", _st, _VP)
_sig("hpsb_context_attach_local", _st, _VP, _VP, ctypes.c_int)
_sig("hpsb_context_comm_info", _st, _VP, _I, _I)
_sig("hpsb_merge_owners", _st, ctypes.c_int, ctypes.c_int, ctypes.c_int, _I)
_sig("hpsb_partition", _st, ctypes.c_int, ctypes.c_int, ctypes.c_int, _I, _I, _I)
_sig("hpsb_hierarchy_pinned_flops", _st, _VP, _D, _D)
_sig("hpsb_precond_pinned_bytes", ctypes.c_double, _VP)


def _check(status: int, allow=(OK,)) -> int:
    if status not in allow:
        raise HpsError(status, _lib.hpsb_last_error().decode())
    return status


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _cplx(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def version() -> str:
    return _lib.hpsb_version().decode()


# ------------------------------------------------------------ host structure
def gll_rule(order: int):
    n = order + 1
    x, w, d = np.zeros(n), np.zeros(n), np.zeros(n * n)
    _check(_lib.hpsb_gll_rule(order, _dp(x), _dp(w), _dp(d)))
    return x, w, d.reshape(n, n, order="F")


def index_sets(order: int) -> dict:
    m, np1 = order - 1, order + 1
    sizes = [m, m, m, m, m * m, np1 * np1 - 4, np1 * np1]
    out = np.zeros(sum(sizes), dtype=np.int32)
    _check(_lib.hpsb_index_sets(order, out.ctypes.data_as(_I)))
    names = ["left", "right", "bottom", "top", "interior", "noncorner", "comp_of_full"]
    res, off = {}, 0
    for name, s in zip(names, sizes):
        res[name] = out[off:off + s].copy()
        off += s
    res["boundary"] = np.concatenate([res["left"], res["right"], res["bottom"], res["top"]])
    return res


def face_graph(n: int) -> dict:
    if n < 2 or n & (n - 1):
        _check(_lib.hpsb_face_graph(n, None, None, None))
    nf, L = 2 * n * (n - 1), 2 * int(np.log2(n))
    faces = np.zeros(6 * nf, dtype=np.int32)
    lr = np.zeros(2 * L, dtype=np.int32)
    foe = np.zeros(4 * n * n, dtype=np.int32)
    _check(_lib.hpsb_face_graph(n, faces.ctypes.data_as(_I), lr.ctypes.data_as(_I),
                                foe.ctypes.data_as(_I)))
    return {"faces": faces.reshape(nf, 6), "level_range": lr.reshape(L, 2),
            "face_of_element": foe.reshape(n * n, 4)}


# ------------------------------------------------------------ problems
@dataclass
class Problem:
    """Sampled problem data (the reference's ProblemSpec evaluated on the mesh)."""
    n: int
    order: int
    kappa: float
    eta: float
    coeff: np.ndarray      # [n^2, (N+1)^2] real, c = kappa^2 (1 - b)
    source: np.ndarray     # [n^2, (N-1)^2] complex, s at interior nodes
    tside: np.ndarray      # [nrhs, n^2, 4, N-1] complex, t on physical sides
    source_zero: bool
    restart: int = 60
    tol: float = 1e-8


def problem(kind: int = 2, config: int = 0, seed: int | None = None, n: int = 0, order: int = 0,
            kappa: float = 0.0) -> Problem:
    """kind 0: ProblemSpec::bump(kappa); 1: ProblemSpec::planewave(kappa); 2: BASELINE config."""
    if seed is None:
        seed = config
    no, oo, nr = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    kk, rs, tl = ctypes.c_double(), ctypes.c_int(), ctypes.c_double()
    _check(_lib.hpsb_problem_dims(kind, config, n, order, ctypes.byref(no), ctypes.byref(oo),
                                  ctypes.byref(nr), ctypes.byref(kk), ctypes.byref(rs),
                                  ctypes.byref(tl)))
    n, order, nrhs = no.value, oo.value, nr.value
    if kind == 2 and not kappa:
        kappa = kk.value  # the config's own wavenumber (else an override)
    ne, np1, m = n * n, order + 1, order - 1
    coeff = np.zeros((ne, np1 * np1))
    source = np.zeros((ne, m * m), dtype=np.complex128)
    tside = np.zeros((nrhs, ne, 4, m), dtype=np.complex128)
    zero = ctypes.c_int()
    _check(_lib.hpsb_problem_sample(kind, config, seed, n, order, kappa, _dp(coeff),
                                    _dp(source.view(np.float64)), _dp(tside.view(np.float64)),
                                    ctypes.byref(zero)))
    return Problem(n, order, kappa, kappa, coeff, source, tside, bool(zero.value),
                   rs.value if kind == 2 else 60, tl.value if kind == 2 else 1e-8)


# ------------------------------------------------------------ objects
class Context:
    """One CUDA device + stream (all objects built from it share the stream)."""

    def __init__(self, device: int = 0):
        h = _VP()
        _check(_lib.hpsb_context_create(device, ctypes.byref(h)))
        self._h = h

    def synchronize(self):
        _check(_lib.hpsb_context_synchronize(self._h))

    @property
    def launches(self) -> int:
        return int(_lib.hpsb_context_launches(self._h))

    def attach_nccl(self, uid: bytes, rank: int, world: int):
        """Shard every object built on this context over `world` GPUs (NCCL)."""
        _check(_lib.hpsb_context_attach_nccl(self._h, uid, rank, world))

    def attach_local(self, group: "LocalGroup", rank: int):
        """Single-process emulation: this context is `rank` of `group`."""
        _check(_lib.hpsb_context_attach_local(self._h, group._h, rank))
        self._group = group

    @property
    def rank_world(self):
        r, w = ctypes.c_int(), ctypes.c_int()
        _check(_lib.hpsb_context_comm_info(self._h, ctypes.byref(r), ctypes.byref(w)))
        return r.value, w.value

    def timer_start(self):
        _check(_lib.hpsb_context_timer_start(self._h))

    def timer_stop(self) -> float:
        s = ctypes.c_double()
        _check(_lib.hpsb_context_timer_stop(self._h, ctypes.byref(s)))
        return s.value

    def profile(self, enable: bool = True):
        _check(_lib.hpsb_context_profile(self._h, int(enable)))

    def profile_reset(self):
        _check(_lib.hpsb_context_profile_reset(self._h))

    def profile_entries(self) -> dict:
        """{kernel: {launches, ms, bytes, flops}} from CUDA events on the context stream."""
        out = {}
        buf = ctypes.create_string_buffer(64)
        for i in range(_lib.hpsb_context_profile_count(self._h)):
            n, ms, b, f = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
            _check(_lib.hpsb_context_profile_entry(self._h, i, buf, 64, ctypes.byref(n),
                                                   ctypes.byref(ms), ctypes.byref(b),
                                                   ctypes.byref(f)))
            out[buf.value.decode()] = {"launches": n.value, "ms": ms.value, "bytes": b.value,
                                       "flops": f.value}
        return out

    def close(self):
        # at interpreter shutdown the module globals may already be cleared
        if getattr(self, "_h", None) and _lib is not None:
            _lib.hpsb_context_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.hpsb_nccl_unique_id(buf))
    return buf.raw


def partition(n: int, world: int, rank: int) -> dict:
    """Host-side sharding plan: element owners, face owners (-1 = shared top level)."""
    nf = 2 * n * (n - 1)
    eo = np.zeros(n * n, dtype=np.int32)
    fo = np.zeros(nf, dtype=np.int32)
    ll = ctypes.c_int()
    _check(_lib.hpsb_partition(n, world, rank, eo.ctypes.data_as(_I), fo.ctypes.data_as(_I),
                               ctypes.byref(ll)))
    return {"elem_owner": eo, "face_owner": fo, "last_local": ll.value}


def merge_owners(n: int, world: int, level: int) -> np.ndarray:
    """Rank that runs each merge (group) of `level` under `world` ranks."""
    faces = face_graph(n)["faces"]
    ng = int(np.max(faces[faces[:, 4] == level][:, 5])) + 1
    out = np.zeros(ng, dtype=np.int32)
    _check(_lib.hpsb_merge_owners(n, world, level, out.ctypes.data_as(_I)))
    return out


class _Handle:
    _destroy = None

    def close(self):
        if getattr(self, "_h", None):
            type(self)._destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


class LocalGroup(_Handle):
    """Single-process group of emulated ranks (one thread + Context each)."""
    _destroy = _lib.hpsb_local_group_destroy

    def __init__(self, world: int):
        h = _VP()
        _check(_lib.hpsb_local_group_create(world, ctypes.byref(h)))
        self._h, self.world = h, world


class ElementRecords(_Handle):
    """The batched element stage: ItI maps T[e] and outgoing sources H[e]."""
    _destroy = _lib.hpsb_elements_destroy

    def __init__(self, ctx: Context, h, n, order, eta):
        self.ctx, self._h, self.n, self.order, self.eta = ctx, h, n, order, eta
        self.m = order - 1
        self.nb = 4 * self.m

    def fallbacks(self) -> int:
        """Elements redone by the pivoted-LU fallback (indefinite L_ii)."""
        c = ctypes.c_int()
        _check(_lib.hpsb_elements_fallbacks(self._h, ctypes.byref(c)))
        return c.value

    def iti(self, e0: int = 0, count: int | None = None):
        count = self.n * self.n - e0 if count is None else count
        T = np.zeros((count, self.nb * self.nb), dtype=np.complex128)
        H = np.zeros((count, self.nb), dtype=np.complex128)
        _check(_lib.hpsb_elements_get(self._h, e0, count, _dp(T.view(np.float64)),
                                      _dp(H.view(np.float64))))
        return T.reshape(count, self.nb, self.nb).transpose(0, 2, 1), H


def build_elements(ctx: Context, prob: Problem) -> ElementRecords:
    """build_elements(mesh, rule) (proj/src/mesh.cpp:36-109) on the GPU."""
    h = _VP()
    coeff = np.ascontiguousarray(prob.coeff, dtype=np.float64)
    src = None if prob.source_zero else _dp(_cplx(prob.source).view(np.float64))
    _check(_lib.hpsb_elements_build(ctx._h, prob.n, prob.order, prob.eta, _dp(coeff), src,
                                    ctypes.byref(h)))
    return ElementRecords(ctx, h, prob.n, prob.order, prob.eta)


class SkeletonSystem(_Handle):
    """assemble_skeleton's system M g = rhs (proj/src/skeleton.cpp:88-137)."""
    _destroy = _lib.hpsb_skeleton_destroy

    def __init__(self, elements: ElementRecords, h, nrhs):
        self.elements, self._h, self.nrhs = elements, h, nrhs
        self.dim = int(_lib.hpsb_skeleton_dim(h))

    def rhs(self, r: int = 0) -> np.ndarray:
        out = np.zeros(self.dim, dtype=np.complex128)
        _check(_lib.hpsb_skeleton_rhs(self._h, r, _dp(out.view(np.float64))))
        return out

    def apply(self, x) -> np.ndarray:
        """BlockMatrix::apply on the skeleton operator."""
        x = _cplx(x)
        y = np.zeros(self.dim, dtype=np.complex128)
        _check(_lib.hpsb_skeleton_apply(self._h, _dp(x.view(np.float64)), _dp(y.view(np.float64))))
        return y

    def rhs_dev_ptr(self, r: int = 0) -> int:
        return int(_lib.hpsb_skeleton_rhs_dev(self._h, r))

    def recover(self, g, r: int = 0) -> np.ndarray:
        """recover_solution (proj/src/problems.cpp:60-92): the field on every
        element's corner-free nodes, shape (n^2, (N+1)^2 - 4)."""
        g = _cplx(g)
        el = self.elements
        field = np.zeros((el.n * el.n, (el.order + 1) ** 2 - 4), dtype=np.complex128)
        _check(_lib.hpsb_recover(self._h, _dp(g.view(np.float64)), r, _dp(field.view(np.float64))))
        return field


def boundary_trace(tside: np.ndarray, n: int) -> np.ndarray:
    """[nrhs, n^2, 4, N-1] element-side data -> [nrhs, 4, n, N-1] physical-side
    data (boundary_side_data order, proj/src/mesh.cpp:111-139): x=0, x=1, y=0,
    y=1, each side's n elements ascending."""
    t = tside.reshape(tside.shape[0], n, n, 4, -1)  # [r, ey, ex, side, k]
    return np.ascontiguousarray(np.stack(
        [t[:, :, 0, 0], t[:, :, n - 1, 1], t[:, 0, :, 2], t[:, n - 1, :, 3]], axis=1))


def assemble_skeleton(elements: ElementRecords, prob: Problem,
                      boundary_only: bool = True) -> SkeletonSystem:
    """assemble_skeleton (proj/src/skeleton.cpp:88-137).  By default only the
    physical-boundary data crosses to the device (hpsb_skeleton_create_boundary);
    boundary_only=False passes the full element-side layout."""
    t = _cplx(prob.tside)
    h = _VP()
    if boundary_only:
        tb = boundary_trace(t, prob.n)
        _check(_lib.hpsb_skeleton_create_boundary(elements._h, _dp(tb.view(np.float64)),
                                                  t.shape[0], ctypes.byref(h)))
    else:
        _check(_lib.hpsb_skeleton_create(elements._h, _dp(t.view(np.float64)), t.shape[0],
                                         ctypes.byref(h)))
    return SkeletonSystem(elements, h, t.shape[0])


class MergeHierarchy(_Handle):
    _destroy = _lib.hpsb_hierarchy_destroy

    def __init__(self, sk: SkeletonSystem, h):
        self.skeleton, self._h = sk, h
        d, t, b, s = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64(), ctypes.c_double()
        _check(_lib.hpsb_hierarchy_info(h, ctypes.byref(d), ctypes.byref(t), ctypes.byref(b),
                                        ctypes.byref(s)))
        self.depth, self.total_levels = d.value, t.value
        self.device_bytes, self.build_seconds = b.value, s.value

    def direct_solve(self, rhs) -> np.ndarray:
        """direct_solve (proj/src/dissection.cpp:240-292); needs a full-depth
        hierarchy built with factor_coarse=True."""
        rhs = _cplx(rhs)
        x = np.zeros_like(rhs)
        _check(_lib.hpsb_direct_solve(self._h, _dp(rhs.view(np.float64)), _dp(x.view(np.float64))))
        return x

    def pinned_flops(self) -> tuple[float, float]:
        """SURVEY §8(d) pinned setup flops: (element stage, merges)."""
        fe, fm = ctypes.c_double(), ctypes.c_double()
        _check(_lib.hpsb_hierarchy_pinned_flops(self._h, ctypes.byref(fe), ctypes.byref(fm)))
        return fe.value, fm.value

    def level_apply(self, level: int, x) -> np.ndarray:
        """y = M_l x on level l's system (faces [first_face(l), total))."""
        x = _cplx(x)
        y = np.zeros_like(x)
        _check(_lib.hpsb_hierarchy_level_apply(self._h, level, _dp(x.view(np.float64)),
                                               _dp(y.view(np.float64))))
        return y

    def level_blocks(self, level: int):
        """(first_face, {(r, c): bs x bs block}) of the level system M_l."""
        nb, ff = ctypes.c_int(), ctypes.c_int()
        _check(_lib.hpsb_hierarchy_level_blocks(self._h, level, ctypes.byref(nb), ctypes.byref(ff),
                                                None, None))
        bs = 2 * self.skeleton.elements.m
        keys = np.zeros(2 * nb.value, dtype=np.int32)
        data = np.zeros(nb.value * bs * bs, dtype=np.complex128)
        _check(_lib.hpsb_hierarchy_level_blocks(self._h, level, ctypes.byref(nb), ctypes.byref(ff),
                                                keys.ctypes.data_as(_I),
                                                _dp(data.view(np.float64))))
        out = {}
        for k in range(nb.value):
            out[(int(keys[2 * k]), int(keys[2 * k + 1]))] = \
                data[k * bs * bs:(k + 1) * bs * bs].reshape(bs, bs, order="F")
        return ff.value, out


def build_hierarchy(sk: SkeletonSystem, depth: int = 0, factor_coarse: bool = True):
    h = _VP()
    _check(_lib.hpsb_hierarchy_build(sk._h, depth, int(factor_coarse), ctypes.byref(h)))
    return MergeHierarchy(sk, h)


class MgPreconditioner(_Handle):
    _destroy = _lib.hpsb_precond_destroy

    def __init__(self, hier: MergeHierarchy, h, cfg: MgConfig):
        self.hierarchy, self._h, self.config = hier, h, cfg

    @property
    def bytes_per_apply(self) -> int:
        """Algorithmic operator bytes one apply streams (the HBM roofline numerator)."""
        return int(_lib.hpsb_precond_bytes(self._h))

    @property
    def pinned_bytes_per_iteration(self) -> float:
        """SURVEY §8(d) pinned operator bytes per outer FGMRES iteration."""
        return float(_lib.hpsb_precond_pinned_bytes(self._h))

    def apply(self, v) -> np.ndarray:
        v = _cplx(v)
        z = np.zeros_like(v)
        _check(_lib.hpsb_precond_apply(self._h, _dp(v.view(np.float64)), _dp(z.view(np.float64))))
        return z


def build_preconditioner(hier: MergeHierarchy, depth: int = 0, gamma: int = 1,
                         coarse_iters: int = 4, exact_coarse: bool = False) -> MgPreconditioner:
    cfg = MgConfig(depth or hier.depth, gamma, coarse_iters, int(exact_coarse))
    h = _VP()
    _check(_lib.hpsb_precond_create(hier._h, cfg, ctypes.byref(h)))
    return MgPreconditioner(hier, h, cfg)


def fgmres(sk: SkeletonSystem, rhs, precond: MgPreconditioner | None, restart: int = 60,
           tol: float = 1e-8, max_iters: int = 2000, record_history: bool = False,
           reorthogonalize: bool = True, right: bool = False):
    """Flexible GMRES (fgmres, proj/src/krylov.cpp:188-192); precond None = gmres.
    right=True: gmres with `precond` as a fixed right preconditioner
    (krylov.cpp:180-186).  reorthogonalize as KrylovConfig (the reference
    driver sets it, driver.cpp:132); False runs one modified Gram-Schmidt pass.
    record_history adds the per-iteration |g_{j+1}| / ||b|| (krylov.cpp:118)."""
    rhs = _cplx(rhs)
    x = np.zeros_like(rhs)
    rep = SolveReport()
    cfg = KrylovConfig(restart, tol, max_iters, int(record_history), int(reorthogonalize))
    fn = _lib.hpsb_gmres if right else _lib.hpsb_fgmres
    _check(fn(sk._h, precond._h if precond else None, _dp(rhs.view(np.float64)),
              _dp(x.view(np.float64)), cfg, ctypes.byref(rep)),
           allow=(OK, NO_CONVERGENCE))
    out = rep.as_dict()
    if record_history:
        ctx = sk.elements.ctx._h
        count = int(_lib.hpsb_context_residual_history(ctx, None, 0))
        hist = np.zeros(max(count, 0))
        if count > 0:
            _lib.hpsb_context_residual_history(ctx, _dp(hist), count)
        out["residual_history"] = hist.tolist()
    return x, out


def fgmres_batch(sk: SkeletonSystem, rhs, precond: MgPreconditioner | None, restart: int = 60,
                 tol: float = 1e-8, max_iters: int = 2000, reorthogonalize: bool = True):
    """R <= 32 right-hand sides (rows of `rhs`) solved in lockstep with
    multi-RHS operator applications; one report per right-hand side."""
    rhs = np.ascontiguousarray(np.atleast_2d(rhs), dtype=np.complex128)
    R = rhs.shape[0]
    x = np.zeros_like(rhs)
    reps = (SolveReport * R)()
    cfg = KrylovConfig(restart, tol, max_iters, 0, int(reorthogonalize))
    _check(_lib.hpsb_fgmres_batch(sk._h, precond._h if precond else None,
                                  _dp(rhs.view(np.float64)), _dp(x.view(np.float64)), R, cfg, reps),
           allow=(OK, NO_CONVERGENCE))
    return x, [r.as_dict() for r in reps]


def gmres(sk: SkeletonSystem, rhs, restart: int = 60, tol: float = 1e-8, max_iters: int = 2000,
          right_precond: MgPreconditioner | None = None, record_history: bool = False,
          reorthogonalize: bool = True):
    """gmres(op, rhs, cfg, right_precond) (proj/src/krylov.cpp:180-186)."""
    return fgmres(sk, rhs, right_precond, restart, tol, max_iters, record_history,
                  reorthogonalize, right=True)


def merge_pair(ctx: Context, T1, H1, T2, H2, alpha: int, beta: int, side_len: int):
    """merge_pair (proj/src/dissection.cpp:23-82) on the GPU; returns (T_pair, H_pair)."""
    m = side_len
    T1 = np.asfortranarray(T1, dtype=np.complex128).ravel(order="F")
    T2 = np.asfortranarray(T2, dtype=np.complex128).ravel(order="F")
    H1, H2 = _cplx(H1), _cplx(H2)
    T = np.zeros(36 * m * m, dtype=np.complex128)
    H = np.zeros(6 * m, dtype=np.complex128)
    _check(_lib.hpsb_merge_pair(ctx._h, m, _dp(T1.view(np.float64)), _dp(H1.view(np.float64)),
                                _dp(T2.view(np.float64)), _dp(H2.view(np.float64)), alpha, beta,
                                _dp(T.view(np.float64)), _dp(H.view(np.float64))))
    return T.reshape(6 * m, 6 * m, order="F"), H
