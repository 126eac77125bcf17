"""Python face of the B200 correction-step library.

Mirrors the reference's C++ namespace API for the hot path (names and argument
meaning follow /root/reference/proj/include/ksafem/*.hpp) on top of the C-ABI in
include/ksb.h. Host arrays are numpy; device arrays are `DeviceArray`s owned by
a `Context`.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as _N
from ._native import check, lib

MAT_S, MAT_M, MAT_AOP, MAT_USER0 = 0, 1, 2, 8
POT_COULOMB, POT_GAUSSIAN = 0, 1


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_N.DP)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(_N.IP)


# ----------------------------------------------------------------------------- mesh
class Mesh:
    """Host tetrahedral mesh (reference mesh::TetMesh, proj/include/ksafem/mesh.hpp:43-87)."""

    _ARR = {  # what -> (dtype, columns, size index)
        "xyz": (0, np.float64, 3, 0), "tets": (1, np.int32, 4, 1), "tuple": (2, np.int32, 4, 1),
        "tag": (3, np.int8, 1, 1), "parent": (4, np.int32, 1, 1), "vparent": (5, np.int32, 2, 0),
        "on_boundary": (6, np.uint8, 1, 0), "boundary_faces": (7, np.int32, 3, 2),
        "interior_faces": (8, np.int32, 3, 3), "interior_face_tets": (9, np.int32, 2, 3),
        "interior_face_geom": (10, np.float64, 5, 3),
    }

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None):
            lib.ksb_mesh_free(self._h)
            self._h = None

    @staticmethod
    def box(lo, hi, n: int) -> "Mesh":
        """build_box_mesh (proj/src/mesh.cpp:281-331)."""
        lo = np.ascontiguousarray(lo, np.float64)
        hi = np.ascontiguousarray(hi, np.float64)
        h = C.c_void_p()
        check(lib.ksb_mesh_box(_dp(lo), _dp(hi), int(n), C.byref(h)))
        return Mesh(h)

    def uniform_refine(self) -> "Mesh":
        """uniform_refine (proj/src/mesh.cpp:333-343)."""
        h = C.c_void_p()
        check(lib.ksb_mesh_uniform_refine(self._h, C.byref(h)))
        return Mesh(h)

    def adapt_refine(self, marked) -> "Mesh":
        """adapt_refine (proj/src/mesh.cpp:345-368)."""
        m = np.ascontiguousarray(marked, np.int32)
        h = C.c_void_p()
        check(lib.ksb_mesh_adapt_refine(self._h, _ip(m), len(m), C.byref(h)))
        return Mesh(h)

    def save(self, path) -> None:
        """binary dump (include/ksb.h ksb_mesh_save): defining arrays, faces recomputed on load"""
        check(lib.ksb_mesh_save(self._h, str(path).encode()))

    @staticmethod
    def load(path) -> "Mesh":
        h = C.c_void_p()
        check(lib.ksb_mesh_load(str(path).encode(), C.byref(h)))
        return Mesh(h)

    def sizes(self):
        s = (C.c_int64 * 8)()
        check(lib.ksb_mesh_sizes(self._h, s))
        return list(s)

    @property
    def n_vertices(self):
        return self.sizes()[0]

    @property
    def n_tets(self):
        return self.sizes()[1]

    @property
    def level(self):
        return self.sizes()[4]

    def array(self, name: str) -> np.ndarray:
        what, dt, cols, si = self._ARR[name]
        rows = self.sizes()[si]
        out = np.empty((rows, cols) if cols > 1 else (rows,), dt)
        check(lib.ksb_mesh_get(self._h, what, out.ctypes.data_as(C.c_void_p)))
        return out


class Hierarchy:
    """fem::SpaceHierarchy (proj/include/ksafem/fespace.hpp:65-81)."""

    def __init__(self):
        h = C.c_void_p()
        check(lib.ksb_hier_create(C.byref(h)))
        self._h = h
        self.meshes = []

    def __del__(self):
        if getattr(self, "_h", None):
            lib.ksb_hier_free(self._h)
            self._h = None

    def push(self, m: Mesh) -> None:
        check(lib.ksb_hier_push(self._h, m._h))
        self.meshes.append(m)

    @property
    def n_levels(self):
        return lib.ksb_hier_levels(self._h)

    def save(self, path) -> None:
        """binary dump of every level (include/ksb.h ksb_hier_save)"""
        check(lib.ksb_hier_save(self._h, str(path).encode()))

    @staticmethod
    def load(path) -> "Hierarchy":
        h = C.c_void_p()
        check(lib.ksb_hier_load(str(path).encode(), C.byref(h)))
        out = Hierarchy.__new__(Hierarchy)
        out._h = h
        out.meshes = []
        for k in range(lib.ksb_hier_levels(h)):
            m = C.c_void_p()
            check(lib.ksb_hier_mesh(h, k, C.byref(m)))
            out.meshes.append(Mesh(m))
        return out

    def prolongation(self, level: int):
        n = self.meshes[level].n_vertices
        col = np.empty((n, 4), np.int32)
        val = np.empty((n, 4), np.float64)
        check(lib.ksb_hier_prolongation(self._h, level, _ip(col), _dp(val)))
        return col, val


def save_state(path, level: int, lambdas, Phi: np.ndarray, w: np.ndarray, N: int | None = None) -> None:
    """binary solver state of one level (include/ksb.h ksb_state_save): lambdas, interior orbital block, w"""
    lam = np.ascontiguousarray(lambdas, np.float64)
    P = np.ascontiguousarray(Phi, np.float64)
    P2 = P.reshape(P.shape[0], -1)
    wv = np.ascontiguousarray(w, np.float64)
    N = int(N or len(lam))
    check(lib.ksb_state_save(str(path).encode(), int(level), N, P2.shape[0], wv.shape[0], _dp(lam), _dp(P2),
                             P2.shape[1], _dp(wv)))


def load_state(path) -> dict:
    s = (C.c_int64 * 4)()
    check(lib.ksb_state_sizes(str(path).encode(), s))
    level, N, ni, n = (int(x) for x in s)
    lam, Phi, w = np.empty(N), np.empty((ni, N)), np.empty(n)
    check(lib.ksb_state_load(str(path).encode(), _dp(lam), _dp(Phi), N, _dp(w)))
    return {"level": level, "lambdas": lam, "Phi": Phi, "w": w}


# ----------------------------------------------------------------------------- device
class Context:
    """One device, one stream (include/ksb.h ksb_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib.ksb_ctx_create(int(device), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib.ksb_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        check(lib.ksb_ctx_stream(self._h, C.byref(s)))
        return s.value or 0

    def sync(self):
        check(lib.ksb_ctx_sync(self._h))

    def set_profiling(self, on: bool):
        check(lib.ksb_ctx_set_profiling(self._h, int(bool(on))))

    def kernel_time(self, name: str):
        ms = C.c_double()
        cnt = C.c_int64()
        check(lib.ksb_ctx_kernel_time(self._h, name.encode(), C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value

    def launches(self) -> int:
        n = C.c_int64()
        check(lib.ksb_ctx_kernel_launches(self._h, C.byref(n)))
        return n.value

    def reset_counters(self):
        check(lib.ksb_ctx_reset_counters(self._h))

    def empty(self, shape, dtype=np.float64) -> "DeviceArray":
        return DeviceArray(self, shape, dtype)

    def to_device(self, a: np.ndarray) -> "DeviceArray":
        d = DeviceArray(self, a.shape, a.dtype)
        d.upload(a)
        return d


class DeviceArray:
    @classmethod
    def wrap(cls, ctx: Context, ptr: int, shape, dtype=np.float64, keep=None) -> "DeviceArray":
        """non-owning view of device memory allocated elsewhere (e.g. a torch tensor, kept alive by `keep`)"""
        d = cls.__new__(cls)
        d.ctx = ctx
        d.shape = tuple(int(s) for s in (shape if isinstance(shape, (tuple, list)) else (shape,)))
        d.dtype = np.dtype(dtype)
        d.nbytes = int(np.prod(d.shape)) * d.dtype.itemsize
        d.ptr = C.c_void_p(int(ptr))
        d._owned = False
        d._keep = keep
        return d

    def __init__(self, ctx: Context, shape, dtype=np.float64):
        self._owned = True
        self.ctx = ctx
        self.shape = tuple(int(s) for s in (shape if isinstance(shape, (tuple, list)) else (shape,)))
        self.dtype = np.dtype(dtype)
        self.nbytes = int(np.prod(self.shape)) * self.dtype.itemsize
        p = C.c_void_p()
        check(lib.ksb_malloc(ctx._h, C.byref(p), self.nbytes))
        self.ptr = p

    def __del__(self):
        if getattr(self, "_owned", True) and getattr(self, "ptr", None) and getattr(self.ctx, "_h", None):
            lib.ksb_free(self.ctx._h, self.ptr)
        self.ptr = None

    def upload(self, a: np.ndarray):
        a = np.ascontiguousarray(a, self.dtype)
        assert a.nbytes == self.nbytes
        check(lib.ksb_memcpy_h2d(self.ctx._h, self.ptr, a.ctypes.data_as(C.c_void_p), self.nbytes))
        self.ctx.sync()

    def download(self) -> np.ndarray:
        out = np.empty(self.shape, self.dtype)
        check(lib.ksb_memcpy_d2h(self.ctx._h, out.ctypes.data_as(C.c_void_p), self.ptr, self.nbytes))
        self.ctx.sync()
        return out


@dataclass
class SolveStats:
    """fem::SolveStats (proj/include/ksafem/solver.hpp:10-15)."""
    iterations: int
    relative_residual: float
    converged: bool
    breakdown: bool


class Level:
    """Device-resident fine level: FE space split, interior patterns, operators."""

    def __init__(self, ctx: Context, hier: Hierarchy, level: int):
        h = C.c_void_p()
        check(lib.ksb_level_create(ctx._h, hier._h, int(level), C.byref(h)))
        self._h = h
        self.ctx = ctx
        s = (C.c_int64 * 10)()
        check(lib.ksb_level_sizes(self._h, s))
        (self.n, self.ni, self.nb, self.nt, self.nnz_ii, self.nnz_ib, self.nH, self.nct, self.ncv, _) = list(s)

    def close(self):
        if getattr(self, "_h", None):
            lib.ksb_level_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def index(self, what: str) -> np.ndarray:
        spec = {"ii_ptr": (0, np.int32, self.ni + 1), "ii_col": (1, np.int32, self.nnz_ii),
                "ib_ptr": (2, np.int32, self.ni + 1), "ib_col": (3, np.int32, self.nnz_ib),
                "interior": (4, np.int32, self.ni), "pint_col": (5, np.int32, self.ni * 4),
                "pint_val": (6, np.float64, self.ni * 4), "t8_col": (7, np.int32, self.ni * 16), "lo_perm": (8, np.int32, self.ni),
                "lo_ptr": (9, np.int32, self.ni + 1), "lo_col": (10, np.int32, self.nnz_ii),
                "dia": (11, np.int32, 16), "ut_sizes": (12, np.int32, 3), "lo_map": (17, np.int32, self.nnz_ii)}
        if what in ("ut_rows", "ut_eptr", "ut_ent", "ut_map"):
            nt, ne, R = (int(x) for x in self.index("ut_sizes"))
            spec["ut_rows"] = (13, np.int32, nt * R)
            spec["ut_eptr"] = (14, np.int32, nt + 1)
            spec["ut_ent"] = (15, np.int32, ne)
            spec["ut_map"] = (16, np.int32, ne * R)
        spec = spec[what]
        out = np.empty(spec[2], spec[1])
        check(lib.ksb_level_index(self._h, spec[0], out.ctypes.data_as(C.c_void_p)))
        return out

    def assemble(self, mat: int, c_s=0.0, c_m=0.0, potential=None, c_p=1.0, w: DeviceArray | None = None, c_w=1.0):
        """values(mat) = c_s S + c_m M + c_p M_pot + c_w M_w (Keast rule, proj/src/assembly.cpp:109-131).

        potential: (kind, params[n_centers, 4 or 5]) or None.
        """
        if potential is not None:
            kind, params = potential
            params = np.ascontiguousarray(params, np.float64)
            nc = params.shape[0]
            pp = _dp(params.reshape(-1))
        else:
            kind, nc, pp = 0, 0, None
        check(lib.ksb_mat_assemble(self._h, int(mat), float(c_s), float(c_m), int(kind), int(nc), pp,
                                   float(c_p), w.ptr if w is not None else None, float(c_w)))

    def axpby(self, dst: int, a: float, x: int, b: float, y: int):
        check(lib.ksb_mat_axpby(self._h, dst, float(a), x, float(b), y))

    def values(self, mat: int, part: int = 0) -> np.ndarray:
        out = np.empty(self.nnz_ii if part == 0 else self.nnz_ib, np.float64)
        check(lib.ksb_mat_values(self._h, mat, part, _dp(out)))
        return out

    def spmm(self, mat: int, X: DeviceArray, Y: DeviceArray, N: int, ldx: int | None = None, ldy: int | None = None):
        check(lib.ksb_spmm(self._h, mat, X.ptr, int(N), int(ldx or N), Y.ptr, int(ldy or N)))

    @staticmethod
    def cg_options(tol=1e-9, max_iterations=20000, fixed_iterations=0, check_every=8, precond=0) -> _N.CgOpts:
        """precond 0: Jacobi (the fused production CG); 1: the reference's exact SGS (parity runs)"""
        o = _N.CgOpts()
        check(lib.ksb_cg_defaults(C.byref(o)))
        o.tol = tol
        o.max_iterations = max_iterations
        o.fixed_iterations = fixed_iterations
        o.check_every = check_every
        o.precond = precond
        return o

    def cg_solve(self, mat: int, B: DeviceArray, X: DeviceArray, N: int, ld: int | None = None, opts=None,
                 shift_mat: int = -1, sigma=None):
        """Multi-RHS PCG on interior blocks; returns per-column SolveStats."""
        opts = opts or self.cg_options()
        st = (_N.CgStats * N_cols(N))()
        sig = np.ascontiguousarray(sigma, np.float64) if sigma is not None else None
        check(lib.ksb_cg_solve(self._h, mat, shift_mat, _dp(sig) if sig is not None else None, B.ptr, X.ptr,
                               int(N), int(ld or N), C.byref(opts), st))
        return [SolveStats(s.iterations, s.relative_residual, bool(s.converged), bool(s.breakdown)) for s in st]

    def cg_solve_host(self, mat: int, B: np.ndarray, N: int, ld: int | None = None, opts=None, shift_mat=-1,
                      sigma=None, out: np.ndarray | None = None):
        """Same as cg_solve with host buffers (H2D + D2H inside the call)."""
        opts = opts or self.cg_options()
        ld = int(ld or N)
        B = np.ascontiguousarray(B, np.float64)
        X = out if out is not None else np.empty_like(B)
        st = (_N.CgStats * N_cols(N))()
        sig = np.ascontiguousarray(sigma, np.float64) if sigma is not None else None
        check(lib.ksb_cg_solve_host(self._h, mat, shift_mat, _dp(sig) if sig is not None else None,
                                    B.ctypes.data_as(C.c_void_p), X.ctypes.data_as(C.c_void_p), int(N), ld,
                                    C.byref(opts), st))
        return X, [SolveStats(s.iterations, s.relative_residual, bool(s.converged), bool(s.breakdown)) for s in st]


    # ------------------------------------------------------------------ correction step
    XC = {"none": 0, "x_alpha": 1, "lda": 2}

    def set_system(self, atoms, n_pairs=1, occupancy=2.0, xc="lda", alpha=0.77298, exchange_exponent=1.0 / 3.0,
                   hartree=True, xc_on=True):
        """model::MolecularSystem + mode switches (proj/include/ksafem/ks_model.hpp:26-34)."""
        a = np.ascontiguousarray(np.asarray(atoms, np.float64).reshape(-1, 4))
        check(lib.ksb_system_set(self._h, _dp(a.reshape(-1)), a.shape[0], int(n_pairs), float(occupancy),
                                 self.XC[xc], float(alpha), float(exchange_exponent), int(hartree), int(xc_on)))
        self.N = int(n_pairs)
        self.occ = float(occupancy)
        self.xc = (self.XC[xc] if xc_on else 0, float(alpha), float(exchange_exponent))

    def level_ops(self):
        """make_level_ops (proj/src/driver.cpp:35-47)."""
        check(lib.ksb_level_ops(self._h))

    @staticmethod
    def step_options(**kw) -> _N.StepOpts:
        o = _N.StepOpts()
        check(lib.ksb_step_defaults(C.byref(o)))
        for k, v in kw.items():
            setattr(o, k, v)
        return o

    @staticmethod
    def _log(lg, att, its):
        return {"inner_iterations": lg.inner_iterations, "hartree_iterations": lg.hartree_iterations,
                "delta": lg.delta, "ms_bvp": lg.ms_bvp, "ms_hartree": lg.ms_hartree, "ms_project": lg.ms_project,
                "ms_inner": lg.ms_inner, "ms_total": lg.ms_total, "cg_iterations": int(lg.cg_iterations),
                "attempts": att.tolist(), "iterations": its.tolist()}

    def coarse_scf(self, tol=1e-6, max_iterations=200, mixing=0.3, hartree=True, xc=True, tol_eig=1e-9, norm_l1=False):
        """scf::self_consistent_solve on level 0 (proj/src/scf.cpp:22-90): (lambdas, Phi, rho, w, iterations, history)."""
        o = _N.ScfOpts()
        check(lib.ksb_scf_defaults(C.byref(o)))
        o.tol, o.max_iterations, o.mixing = float(tol), int(max_iterations), float(mixing)
        o.hartree_on, o.xc_on, o.tol_eig = int(hartree), int(xc), float(tol_eig)
        o.norm_l1 = int(norm_l1)
        N = self.N
        ld = N if N == 1 else N + (N & 1)
        lam = np.empty(N)
        Phi = self.ctx.empty((self.ni, ld))
        rho, w = self.ctx.empty((self.n,)), self.ctx.empty((self.n,))
        it = C.c_int()
        hist = np.zeros(max(1, int(max_iterations)))
        st = lib.ksb_coarse_scf(self._h, C.byref(o), _dp(lam), Phi.ptr, ld, rho.ptr, w.ptr, C.byref(it), _dp(hist),
                                len(hist))
        self.last_scf_history = hist[:it.value].copy()  # kept when the iteration fails (the error is raised below)
        check(st)
        return lam, Phi, rho, w, it.value, hist[:it.value]

    def correction_step(self, lambdas: np.ndarray, Phi: DeviceArray, w: DeviceArray, ld: int | None = None, **opts):
        """One outer iteration (proj/src/driver.cpp:106-150) on device-resident state; lambdas updated in place."""
        o = self.step_options(**opts)
        lg = _N.StepLog()
        att = np.zeros(self.N, np.int32)
        its = np.zeros(self.N, np.int32)
        check(lib.ksb_correction_step(self._h, C.byref(o), _dp(lambdas), Phi.ptr, int(ld or Phi.shape[1]), w.ptr,
                                      C.byref(lg), _ip(att), _ip(its)))
        return self._log(lg, att, its)

    def mlc_begin(self, lambdas: np.ndarray, Phi: DeviceArray, w: DeviceArray, **opts):
        """standard MLC setup (proj/src/driver.cpp:206-243): orbital BVPs with the warm potentials, Hartree bc"""
        o = self.step_options(**opts)
        lg = _N.StepLog()
        att = np.zeros(self.N, np.int32)
        its = np.zeros(self.N, np.int32)
        check(lib.ksb_mlc_begin(self._h, C.byref(o), _dp(np.ascontiguousarray(lambdas, np.float64)), Phi.ptr,
                                int(Phi.shape[1]), w.ptr, C.byref(lg), _ip(att), _ip(its)))
        return self._log(lg, att, its)

    def mlc_sweep(self, lambdas: np.ndarray, Phi: DeviceArray, **opts) -> float:
        """one correction-space sweep (proj/src/driver.cpp:244-300); lambdas and Phi updated, returns the H1 change"""
        o = self.step_options(**opts)
        d = C.c_double()
        check(lib.ksb_mlc_sweep(self._h, C.byref(o), _dp(lambdas), Phi.ptr, int(Phi.shape[1]), C.byref(d)))
        return d.value

    def mlc_finish(self, w: DeviceArray, rho: DeviceArray | None = None, **opts):
        o = self.step_options(**opts)
        check(lib.ksb_mlc_finish(self._h, C.byref(o), w.ptr, rho.ptr if rho is not None else None))

    def correction_step_host(self, lambdas: np.ndarray, Phi: np.ndarray, w: np.ndarray, **opts):
        o = self.step_options(**opts)
        lg = _N.StepLog()
        att = np.zeros(self.N, np.int32)
        its = np.zeros(self.N, np.int32)
        check(lib.ksb_correction_step_host(self._h, C.byref(o), _dp(lambdas), Phi.ctypes.data_as(C.c_void_p),
                                           int(Phi.shape[1]), w.ctypes.data_as(C.c_void_p), C.byref(lg), _ip(att),
                                           _ip(its)))
        return self._log(lg, att, its)

    def density_xc(self, Phi: DeviceArray, rho: DeviceArray, vxc: DeviceArray | None = None, N=None, ld=None):
        check(lib.ksb_density_xc(self._h, Phi.ptr, int(N or self.N), int(ld or Phi.shape[1]), rho.ptr,
                                 vxc.ptr if vxc is not None else None))

    def xc_field(self, rho: DeviceArray, vxc: DeviceArray):
        """model::xc_potential_field (proj/src/ks_model.cpp:101-105) with the level's functional."""
        kind, alpha, p = self.xc
        check(lib.ksb_xc_field(self._h, kind, alpha, p, rho.ptr, vxc.ptr))

    def density(self, Phi: DeviceArray, rho: DeviceArray, N=None, ld=None):
        check(lib.ksb_density(self._h, Phi.ptr, int(N or self.N), int(ld or Phi.shape[1]), self.occ, rho.ptr))

    def moments(self, rho: DeviceArray) -> np.ndarray:
        out = np.empty(16)
        check(lib.ksb_moments(self._h, rho.ptr, _dp(out)))
        return out

    def boundary_values(self, moments: np.ndarray, bcb: DeviceArray):
        m = np.ascontiguousarray(moments, np.float64)
        check(lib.ksb_boundary_values(self._h, _dp(m), bcb.ptr))

    def prolong(self, src: DeviceArray, dst: DeviceArray, src_interior: bool, dst_interior: bool, ncols=None):
        """fem::SpaceHierarchy::prolong from the previous level (proj/src/fespace.cpp:76-84), bit-exact:
        src on level-1 (full vertex rows or interior block), dst on this level (full or interior block)."""
        sc = src.shape[1] if len(src.shape) > 1 else 1
        dc = dst.shape[1] if len(dst.shape) > 1 else 1
        check(lib.ksb_prolong(self._h, src.ptr, int(src_interior), sc, int(ncols or min(sc, dc)), dst.ptr,
                              int(dst_interior), dc))

    def sqload(self, Phi: DeviceArray, out: DeviceArray, N=None, ld=None):
        check(lib.ksb_sqload(self._h, Phi.ptr, int(N or self.N), int(ld or Phi.shape[1]), out.ptr))

    def hartree_solve(self, Phi: DeviceArray, bcb: DeviceArray, w: DeviceArray, tol=1e-9, N=None, ld=None):
        it = C.c_int()
        check(lib.ksb_hartree_solve(self._h, Phi.ptr, int(N or self.N), int(ld or Phi.shape[1]), bcb.ptr, float(tol),
                                    w.ptr, C.byref(it)))
        return it.value

    def outer_solve(self, w_hat: DeviceArray, vxc: DeviceArray, lambdas, Phi: DeviceArray, PhiT: DeviceArray, **opts):
        o = self.step_options(**opts)
        lam = np.ascontiguousarray(lambdas, np.float64)
        att = np.zeros(self.N, np.int32)
        its = np.zeros(self.N, np.int32)
        md = C.c_double()
        check(lib.ksb_outer_solve(self._h, C.byref(o), w_hat.ptr, vxc.ptr, _dp(lam), Phi.ptr, int(Phi.shape[1]),
                                  PhiT.ptr, _ip(att), _ip(its), C.byref(md)))
        return att, its, md.value

    def prepare_blocks(self, PhiT: DeviceArray, wt: DeviceArray, ell: DeviceArray, vxc: DeviceArray):
        check(lib.ksb_prepare_blocks(self._h, PhiT.ptr, int(PhiT.shape[1]), wt.ptr, ell.ptr, vxc.ptr))

    BLOCKS = {"A_H1": 0, "A_H3": 1, "A_H4": 2, "M_H": 3, "C_H": 4, "d_Hh": 5, "lift_load": 6, "scalars": 7,
              "A_h4": 10, "b_H1": 11, "b_H3": 12, "b_H4": 13, "rhs": 14, "c_Hh": 15, "d_phi": 16, "beta1": 17,
              "beta3": 18, "beta4": 19, "gamma": 20, "zeta_phi": 21}

    def blocks(self, name: str) -> np.ndarray:
        w = self.BLOCKS[name]
        nh, N = self.nH, self.N
        shape = {0: (nh, nh), 1: (nh, nh), 2: (nh, nh), 3: (nh, nh), 4: (nh, nh), 5: (nh,), 6: (nh,), 7: (2,),
                 10: (N, nh, nh)}.get(w, (N, nh) if w < 17 else (N,))
        out = np.empty(int(np.prod(shape)))
        check(lib.ksb_blocks_get(self._h, w, _dp(out)))
        return out.reshape(shape)

    def inner_scf(self, lambdas, **opts):
        o = self.step_options(**opts)
        N, nh = self.N, self.nH
        lam0 = np.ascontiguousarray(lambdas, np.float64)
        lam = np.empty(N)
        phi = np.empty((N, nh))
        th2 = np.empty(N)
        wH = np.empty(nh)
        th1 = C.c_double()
        it = C.c_int()
        cap = max(o.max_inner, o.fixed_sweeps)
        hist = np.zeros(cap)
        check(lib.ksb_inner_scf(self._h, C.byref(o), _dp(lam0), _dp(lam), _dp(phi), _dp(th2), _dp(wH), C.byref(th1),
                                C.byref(it), _dp(hist), cap))
        return dict(lambda_=lam, phi_H=phi, theta2=th2, w_H=wH, theta1=th1.value, iterations=it.value,
                    history=hist[:it.value])

    def expand(self, PhiT: DeviceArray, wt: DeviceArray, bcb: DeviceArray, Phi: DeviceArray, w: DeviceArray):
        check(lib.ksb_expand(self._h, PhiT.ptr, int(PhiT.shape[1]), wt.ptr, bcb.ptr, Phi.ptr, w.ptr))

    def indicators(self, lambdas, Phi: DeviceArray, w: DeviceArray, vxc: DeviceArray, ld: int | None = None):
        """est::compute_indicators (proj/src/estimator.cpp:11-85) on the device: (eta_sq per tet, total)."""
        lam = np.ascontiguousarray(lambdas, np.float64)
        eta = self.ctx.empty((self.nt,))
        tot = C.c_double()
        check(lib.ksb_indicators(self._h, _dp(lam), Phi.ptr, int(ld or Phi.shape[1]), w.ptr, vxc.ptr, eta.ptr,
                                 C.byref(tot)))
        return eta.download(), tot.value

    def norms(self, f: DeviceArray) -> np.ndarray:
        out = np.empty(3)
        check(lib.ksb_norms(self._h, f.ptr, _dp(out)))
        return out

    def l1_norm(self, f: DeviceArray) -> float:
        """fem::l1_norm (proj/src/assembly.cpp:289-291) of a full-length nodal function"""
        out = C.c_double()
        check(lib.ksb_l1_norm(self._h, f.ptr, C.byref(out)))
        return out.value

    def energy(self, Phi: DeviceArray, w: DeviceArray, N=None, ld=None) -> np.ndarray:
        out = np.empty(5)
        check(lib.ksb_energy(self._h, Phi.ptr, int(N or self.N), int(ld or Phi.shape[1]), w.ptr, _dp(out)))
        return out


def dorfler_mark(eta, total_sq: float, theta: float) -> np.ndarray:
    """est::dorfler_mark (proj/src/estimator.cpp:87-104), host side of the C-ABI."""
    e = np.ascontiguousarray(eta, np.float64)
    out = np.empty(len(e), np.int32)
    n = C.c_int64()
    check(lib.ksb_dorfler_mark(_dp(e), len(e), float(total_sq), float(theta), _ip(out), C.byref(n)))
    return out[:n.value].copy()


def N_cols(n: int) -> int:
    return max(1, int(n))
