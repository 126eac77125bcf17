"""ctypes binding of oracle/_build/liboracle.so (TEST INFRASTRUCTURE ONLY)."""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB = _HERE / "_build" / "liboracle.so"


def _load():
    if not LIB.exists():
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return C.CDLL(str(LIB))


lib = _load()
P, PP, I, I64, D = C.c_void_p, C.POINTER(C.c_void_p), C.c_int, C.c_int64, C.c_double
DP, IP, I64P = C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_int64)

_PROTO = {
    "orc_last_error": (C.c_char_p, []),
    "orc_mesh_box": (I, [DP, DP, I, PP]),
    "orc_mesh_uniform": (I, [P, PP]),
    "orc_mesh_adapt": (I, [P, IP, I64, PP]),
    "orc_mesh_free": (None, [P]),
    "orc_mesh_sizes": (I, [P, I64P]),
    "orc_mesh_get": (I, [P, I, P]),
    "orc_mesh_conforming": (I, [P]),
    "orc_mesh_total_volume": (I, [P, DP]),
    "orc_problem_create": (I, [DP, I, I, D, I, D, D, I, I, PP]),
    "orc_problem_free": (None, [P]),
    "orc_problem_push": (I, [P, P]),
    "orc_level_sizes": (I, [P, I, I64P]),
    "orc_interior": (I, [P, I, IP]),
    "orc_prolongation": (I, [P, I, IP, DP]),
    "orc_operator_build": (I, [P, I, D, D, I, I, DP, D, DP, D, I, PP]),
    "orc_operator_free": (None, [P]),
    "orc_operator_nnz": (I, [P, I64P]),
    "orc_operator_ii": (I, [P, IP, IP, DP]),
    "orc_operator_ib": (I, [P, IP, IP, DP]),
    "orc_operator_full": (I, [P, IP, IP, DP]),
    "orc_operator_solve": (I, [P, DP, DP, D, I, DP, IP, DP]),
    "orc_keast": (I, [DP, DP]),
    "orc_prolongation_nnz": (I, [P, I, I, I64P]),
    "orc_prolongation_csc": (I, [P, I, I, IP, IP, DP]),
    "orc_load_nodal": (I, [P, I, DP, DP]),
    "orc_operator_min_diag": (I, [P, DP]),
    "orc_operator_spmv": (I, [P, DP, DP]),
    "orc_operator_pcg": (I, [P, DP, DP, I, D, I, I, IP, DP]),
    "orc_level_matrix": (I, [P, I, I, I, IP, IP, DP]),
    "orc_density": (I, [DP, I, I, D, DP]),
    "orc_xc_potential": (I, [P, DP, I, DP]),
    "orc_xc_energy_density": (I, [P, DP, I, DP]),
    "orc_moments": (I, [P, I, DP, DP]),
    "orc_boundary_values": (I, [P, I, DP, DP]),
    "orc_sqload": (I, [P, I, DP, I, DP]),
    "orc_hartree_exact": (I, [P, I, DP, I, DP, D, DP, IP]),
    "orc_energy": (I, [P, I, DP, I, DP, DP]),
    "orc_indicators": (I, [P, I, DP, DP, I, DP, DP, DP, DP]),
    "orc_last_scf_rho": (I, [P, DP]),
    "orc_last_scf_history": (I, [P, DP, IP]),
    "orc_dorfler": (I, [DP, I64, D, D, IP, C.POINTER(C.c_int64)]),
    "orc_norms": (I, [P, I, DP, DP]),
    "orc_l1_norm": (I, [P, I, DP, DP]),
    "orc_prolong_vec": (I, [P, I, I, DP, I, DP]),
    "orc_coarse_scf": (I, [P, D, I, D, D, DP, DP, DP, IP]),
    "orc_correction_step": (I, [P, I, DP, IP, DP, DP, DP, IP, DP]),
    "orc_solve_level_mlc": (I, [P, I, DP, IP, D, I, DP, DP, DP, DP, IP, DP, I]),
    "orc_outer_solve": (I, [P, I, DP, DP, DP, DP, D, I, DP, IP, IP, DP]),
    "orc_prepare_blocks": (I, [P, I, DP, DP, DP, DP, I, PP]),
    "orc_blocks_free": (None, [P]),
    "orc_blocks_get": (I, [P, I, DP]),
    "orc_inner_scf": (I, [P, DP, D, I, D, I, DP, DP, DP, DP, DP, IP, DP, I]),
    "orc_expand_last": (I, [P, DP, DP]),
    "orc_blocks_f_g": (I, [P, DP, DP, DP, D, DP, DP, DP]),
    "orc_gen_eig": (I, [I, DP, DP, DP, DP]),
    "orc_solve_bordered": (I, [I, DP, DP, DP, D, DP, D, I, D, DP, DP, DP, DP]),
}
for _n, (_r, _a) in _PROTO.items():
    _f = getattr(lib, _n)
    _f.restype = _r
    _f.argtypes = _a

CODES = {1: "nonconvergence", 2: "mismatched-spaces", 3: "singular-quadrature", 4: "ambiguous-selection",
         5: "internal", 6: "invalid-argument", 7: "invalid-domain", 8: "hierarchy"}


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        self.code = CODES.get(status, "unknown")
        super().__init__(f"{self.code}: {msg}")


def _chk(st):
    if st != 0:
        raise OracleError(st, lib.orc_last_error().decode())


def dp(a):
    return None if a is None else a.ctypes.data_as(DP)


def ip(a):
    return a.ctypes.data_as(IP)


def f64(a):
    return np.ascontiguousarray(a, np.float64)


class OMesh:
    ARR = {"xyz": (0, np.float64, 3, 0), "tets": (1, np.int32, 4, 1), "tuple": (2, np.int32, 4, 1),
           "tag": (3, np.int8, 1, 1), "parent": (4, np.int32, 1, 1), "vparent": (5, np.int32, 2, 0),
           "on_boundary": (6, np.uint8, 1, 0), "boundary_faces": (7, np.int32, 3, 2),
           "interior_faces": (8, np.int32, 3, 3), "interior_face_tets": (9, np.int32, 2, 3)}

    def __init__(self, h):
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.orc_mesh_free(self._h)

    @staticmethod
    def box(lo, hi, n):
        h = C.c_void_p()
        _chk(lib.orc_mesh_box(dp(f64(lo)), dp(f64(hi)), n, C.byref(h)))
        return OMesh(h)

    def uniform_refine(self):
        h = C.c_void_p()
        _chk(lib.orc_mesh_uniform(self._h, C.byref(h)))
        return OMesh(h)

    def adapt_refine(self, marks):
        m = np.ascontiguousarray(marks, np.int32)
        h = C.c_void_p()
        _chk(lib.orc_mesh_adapt(self._h, ip(m), len(m), C.byref(h)))
        return OMesh(h)

    def sizes(self):
        s = (C.c_int64 * 8)()
        _chk(lib.orc_mesh_sizes(self._h, s))
        return list(s)

    def array(self, name):
        what, dt, cols, si = self.ARR[name]
        rows = self.sizes()[si]
        out = np.empty((rows, cols) if cols > 1 else (rows,), dt)
        _chk(lib.orc_mesh_get(self._h, what, out.ctypes.data_as(C.c_void_p)))
        return out

    def conforming(self):
        return bool(lib.orc_mesh_conforming(self._h))

    def total_volume(self):
        v = C.c_double()
        _chk(lib.orc_mesh_total_volume(self._h, C.byref(v)))
        return v.value


class Oracle:
    """A system + mesh hierarchy on the CPU oracle (restates proj/src/driver.cpp's level pieces)."""

    def __init__(self, atoms, n_pairs=1, occ=2.0, xc="lda", alpha=0.77298, p_exch=1.0 / 3.0, hartree=True,
                 xc_on=True):
        a = f64(np.asarray(atoms, np.float64).reshape(-1, 4))
        kind = {"none": 0, "x_alpha": 1, "lda": 2}[xc]
        h = C.c_void_p()
        _chk(lib.orc_problem_create(dp(a.reshape(-1)), a.shape[0], n_pairs, occ, kind, alpha, p_exch, int(hartree),
                                    int(xc_on), C.byref(h)))
        self._h = h
        self.N = n_pairs
        self.occ = occ
        self.meshes = []

    def __del__(self):
        if getattr(self, "_h", None):
            lib.orc_problem_free(self._h)

    def push(self, m: OMesh):
        _chk(lib.orc_problem_push(self._h, m._h))
        self.meshes.append(m)

    def sizes(self, level):
        s = (C.c_int64 * 8)()
        _chk(lib.orc_level_sizes(self._h, level, s))
        return list(s)

    def n(self, level):
        return self.meshes[level].sizes()[0]

    def interior(self, level):
        ni = self.sizes(level)[1]
        out = np.empty(ni, np.int32)
        _chk(lib.orc_interior(self._h, level, ip(out)))
        return out

    def prolongation(self, level):
        n = self.n(level)
        col = np.empty((n, 4), np.int32)
        val = np.empty((n, 4), np.float64)
        _chk(lib.orc_prolongation(self._h, level, ip(col), dp(val)))
        return col, val

    def level_matrix(self, level, which, part=0):
        """interior block (part 0) or interior x boundary block (part 1) of S (0), M (1), a_op (2): CSC arrays"""
        s = self.sizes(level)
        ni, nnz = s[1], s[4] if part == 0 else s[5]
        ptr = np.empty(ni + 1 if part == 0 else s[2] + 1, np.int32)
        # CSC of A_ib has boundary columns; sizes unknown up front -> query via operator path instead
        idx = np.empty(nnz, np.int32)
        val = np.empty(nnz, np.float64)
        _chk(lib.orc_level_matrix(self._h, level, which, part, ip(ptr), ip(idx), dp(val)))
        return ptr, idx, val

    def operator(self, level, c_s=0.0, c_m=0.0, potential=None, c_p=1.0, w=None, c_w=1.0, precond=0):
        if potential is not None:
            kind, params = potential
            params = f64(params).reshape(-1)
            nc = len(params) // (4 if kind == 0 else 5)
        else:
            kind, params, nc = 0, None, 0
        h = C.c_void_p()
        _chk(lib.orc_operator_build(self._h, level, c_s, c_m, kind, nc, dp(params), c_p,
                                    dp(f64(w)) if w is not None else None, c_w, precond, C.byref(h)))
        return OOperator(h)

    # physics ------------------------------------------------------------------------------
    def density(self, orb):
        orb = f64(orb)
        n, N = orb.shape
        rho = np.empty(n)
        _chk(lib.orc_density(dp(orb), n, N, self.occ, dp(rho)))
        return rho

    def xc_potential(self, rho):
        rho = f64(rho)
        out = np.empty_like(rho)
        _chk(lib.orc_xc_potential(self._h, dp(rho), len(rho), dp(out)))
        return out

    def xc_energy_density(self, rho):
        rho = f64(rho)
        out = np.empty_like(rho)
        _chk(lib.orc_xc_energy_density(self._h, dp(rho), len(rho), dp(out)))
        return out

    def moments(self, level, rho):
        out = np.empty(16)
        _chk(lib.orc_moments(self._h, level, dp(f64(rho)), dp(out)))
        return out

    def boundary_values(self, level, mom):
        bc = np.empty(self.n(level))
        _chk(lib.orc_boundary_values(self._h, level, dp(f64(mom)), dp(bc)))
        return bc

    def sqload(self, level, orb):
        orb = f64(orb)
        out = np.empty(self.n(level))
        _chk(lib.orc_sqload(self._h, level, dp(orb), orb.shape[1], dp(out)))
        return out

    def hartree_exact(self, level, orb, bc, tol=1e-9):
        orb = f64(orb)
        w = np.empty(self.n(level))
        it = C.c_int()
        _chk(lib.orc_hartree_exact(self._h, level, dp(orb), orb.shape[1], dp(f64(bc)) if bc is not None else None,
                                   tol, dp(w), C.byref(it)))
        return w, it.value

    def energy(self, level, orb, w):
        orb = f64(orb)
        out = np.empty(5)
        _chk(lib.orc_energy(self._h, level, dp(orb), orb.shape[1], dp(f64(w)), dp(out)))
        return out

    def indicators(self, level, lambdas, orb, w, vxc):
        """est::compute_indicators (proj/src/estimator.cpp:11-85): (eta_sq per tet, total)"""
        orb = f64(orb)
        if orb.ndim == 1:
            orb = orb[:, None]
        eta = np.empty(self.meshes[level].sizes()[1])
        tot = C.c_double()
        _chk(lib.orc_indicators(self._h, level, dp(f64(lambdas)), dp(orb), orb.shape[1], dp(f64(w)), dp(f64(vxc)),
                                dp(eta), C.byref(tot)))
        return eta, tot.value

    def norms(self, level, f):
        out = np.empty(3)
        _chk(lib.orc_norms(self._h, level, dp(f64(f)), dp(out)))
        return out

    def l1_norm(self, level, f):
        out = C.c_double()
        _chk(lib.orc_l1_norm(self._h, level, dp(f64(f)), C.byref(out)))
        return out.value

    def prolongation_matrix(self, frm, to):
        import scipy.sparse as sp
        nnz = C.c_int64()
        _chk(lib.orc_prolongation_nnz(self._h, frm, to, C.byref(nnz)))
        nc = self.n(frm)
        ptr = np.empty(nc + 1, np.int32)
        idx = np.empty(nnz.value, np.int32)
        val = np.empty(nnz.value)
        _chk(lib.orc_prolongation_csc(self._h, frm, to, ip(ptr), ip(idx), dp(val)))
        return sp.csc_matrix((val, idx, ptr), shape=(self.n(to), nc))

    def load_nodal(self, level, f):
        out = np.empty(self.n(level))
        _chk(lib.orc_load_nodal(self._h, level, dp(f64(f)), dp(out)))
        return out

    def prolong(self, vec, frm, to):
        v = f64(vec)
        if v.ndim == 1:
            v = v[:, None]
        out = np.empty((self.n(to), v.shape[1]))
        _chk(lib.orc_prolong_vec(self._h, frm, to, dp(v), v.shape[1], dp(out)))
        return out

    def coarse_scf(self, tol=1e-6, max_it=200, mixing=0.3, tol_eig=1e-9):
        n0 = self.n(0)
        lam = np.empty(self.N)
        orb = np.empty((n0, self.N))
        w = np.empty(n0)
        it = C.c_int()
        _chk(lib.orc_coarse_scf(self._h, tol, max_it, mixing, tol_eig, dp(lam), dp(orb), dp(w), C.byref(it)))
        return lam, orb, w, it.value

    def last_scf_history(self):
        """H1 density change per coarse-SCF iteration of the last coarse_scf call, also after it failed"""
        cap = C.c_int(100000)
        buf = np.empty(cap.value)
        _chk(lib.orc_last_scf_history(self._h, dp(buf), C.byref(cap)))
        return buf[:cap.value].copy()

    def last_scf_rho(self):
        """mixed density of the last coarse_scf (ScfResult::rho, proj/src/scf.cpp:73)"""
        out = np.empty(self.n(0))
        _chk(lib.orc_last_scf_rho(self._h, dp(out)))
        return out

    def correction_step(self, level, lambdas, orb, w, tol_linear=1e-9, tol_inner=1e-8, score_floor=1e-8,
                        max_inner=400, nev_pad=4, precond=0, fixed_sweeps=0):
        lam = f64(lambdas).copy()
        orb = f64(orb).copy()
        w = f64(w).copy()
        cd = np.array([tol_linear, tol_inner, score_floor])
        ci = np.array([max_inner, nev_pad, precond, fixed_sweeps], np.int32)
        li = np.zeros(2 + 2 * self.N, np.int32)
        ld = np.zeros(6)
        _chk(lib.orc_correction_step(self._h, level, dp(cd), ip(ci), dp(lam), dp(orb), dp(w), ip(li), dp(ld)))
        log = {"inner_iterations": int(li[0]), "hartree_iterations": int(li[1]),
               "attempts": li[2:2 + self.N].tolist(), "cg_iterations": li[2 + self.N:].tolist(),
               "delta": ld[0], "t_bvp": ld[1], "t_hartree": ld[2], "t_blocks": ld[3], "t_inner": ld[4],
               "t_total": ld[5]}
        return lam, orb, w, log

    def solve_level_mlc(self, level, lambdas, orb, w, tol_outer=1e-6, max_scf=200, tol_linear=1e-9, tol_inner=1e-8,
                        score_floor=1e-8, max_inner=400, nev_pad=4, precond=0):
        """driver::solve_level_mlc (proj/src/driver.cpp:200-302): (lambdas, orbitals, w, rho, deltas)"""
        lam = f64(lambdas).copy()
        orb = f64(orb).copy()
        w = f64(w).copy()
        rho = np.empty(self.n(level))
        cd = np.array([tol_linear, tol_inner, score_floor])
        ci = np.array([max_inner, nev_pad, precond], np.int32)
        sw = C.c_int()
        ds = np.zeros(max(1, max_scf))
        _chk(lib.orc_solve_level_mlc(self._h, level, dp(cd), ip(ci), float(tol_outer), int(max_scf), dp(lam), dp(orb),
                                     dp(w), dp(rho), C.byref(sw), dp(ds), len(ds)))
        return lam, orb, w, rho, ds[:sw.value]

    def outer_solve(self, level, w_hat, vxc, lambdas, orb, tol=1e-9, precond=0):
        n = self.n(level)
        out = np.empty((n, self.N))
        att = np.empty(self.N, np.int32)
        its = np.empty(self.N, np.int32)
        sig = np.empty(4)
        _chk(lib.orc_outer_solve(self._h, level, dp(f64(w_hat)), dp(f64(vxc)), dp(f64(lambdas)), dp(f64(orb)), tol,
                                 precond, dp(out), ip(att), ip(its), dp(sig)))
        return out, att, its, sig

    def prepare_blocks(self, level, phi_tilde, w_tilde, vxc, bc, hartree_on=True):
        h = C.c_void_p()
        _chk(lib.orc_prepare_blocks(self._h, level, dp(f64(phi_tilde)), dp(f64(w_tilde)), dp(f64(vxc)),
                                    dp(f64(bc)) if bc is not None else None, int(hartree_on), C.byref(h)))
        return OBlocks(h, self.N, self.sizes(level)[6], self.n(level))


class OOperator:
    def __init__(self, h):
        self._h = h
        s = (C.c_int64 * 5)()
        _chk(lib.orc_operator_nnz(self._h, s))
        self.nnz_ii, self.nnz_ib, self.ni, self.nnz_full, self.n = list(s)

    def full(self):
        """full n x n matrix as scipy CSC"""
        import scipy.sparse as sp
        ptr = np.empty(self.n + 1, np.int32)
        idx = np.empty(self.nnz_full, np.int32)
        val = np.empty(self.nnz_full)
        _chk(lib.orc_operator_full(self._h, ip(ptr), ip(idx), dp(val)))
        return sp.csc_matrix((val, idx, ptr), shape=(self.n, self.n))

    def solve(self, b, bc=None, tol=1e-9, maxit=20000):
        x = np.empty(self.n)
        st = np.empty(3, np.int32)
        rel = C.c_double()
        _chk(lib.orc_operator_solve(self._h, dp(f64(b)), dp(f64(bc)) if bc is not None else None, tol, maxit, dp(x),
                                    ip(st), C.byref(rel)))
        return x, dict(iterations=int(st[0]), converged=bool(st[1]), breakdown=bool(st[2]),
                       relative_residual=rel.value)

    def __del__(self):
        if getattr(self, "_h", None):
            lib.orc_operator_free(self._h)

    def ii(self):
        ptr = np.empty(self.ni + 1, np.int32)
        idx = np.empty(self.nnz_ii, np.int32)
        val = np.empty(self.nnz_ii)
        _chk(lib.orc_operator_ii(self._h, ip(ptr), ip(idx), dp(val)))
        return ptr, idx, val

    def min_diag(self):
        d = C.c_double()
        _chk(lib.orc_operator_min_diag(self._h, C.byref(d)))
        return d.value

    def spmv(self, x):
        y = np.empty(self.ni)
        _chk(lib.orc_operator_spmv(self._h, dp(f64(x)), dp(y)))
        return y

    def pcg(self, B, tol=1e-9, maxit=20000, fixed=0):
        B = f64(B)
        if B.ndim == 1:
            B = B[:, None]
        N = B.shape[1]
        X = np.empty_like(B)
        st = np.empty(3 * N, np.int32)
        rel = np.empty(N)
        _chk(lib.orc_operator_pcg(self._h, dp(B), dp(X), N, tol, maxit, fixed, ip(st), dp(rel)))
        stats = [dict(iterations=int(st[3 * j]), converged=bool(st[3 * j + 1]), breakdown=bool(st[3 * j + 2]),
                      relative_residual=float(rel[j])) for j in range(N)]
        return X, stats


class OBlocks:
    NAMES = {"A_H1": 0, "A_H3": 1, "A_H4": 2, "M_H": 3, "C_H": 4, "d_Hh": 5, "lift_load": 6, "scalars": 7,
             "hartree_u": 8, "A_h4": 10, "b_H1": 11, "b_H3": 12, "b_H4": 13, "rhs": 14, "c_Hh": 15, "d_phi": 16,
             "beta1": 17, "beta3": 18, "beta4": 19, "gamma": 20, "zeta_phi": 21}

    def __init__(self, h, N, nh, n):
        self._h, self.N, self.nh, self.n = h, N, nh, n

    def __del__(self):
        if getattr(self, "_h", None):
            lib.orc_blocks_free(self._h)

    def get(self, name):
        w = self.NAMES[name]
        nh, N = self.nh, self.N
        shape = {0: (nh, nh), 1: (nh, nh), 2: (nh, nh), 3: (nh, nh), 4: (nh, nh), 5: (nh,), 6: (nh,), 7: (3,),
                 8: (nh,), 10: (N, nh, nh)}.get(w, (N, nh) if w < 17 else (N,))
        out = np.empty(int(np.prod(shape)))
        _chk(lib.orc_blocks_get(self._h, w, dp(out)))
        if w in (0, 1, 2, 3, 4):
            return out.reshape(nh, nh, order="F")
        if w == 10:
            return out.reshape(N, nh, nh).transpose(0, 2, 1)
        return out.reshape(shape)

    def inner_scf(self, lambdas, tol=1e-8, max_it=400, floor=1e-8, pad=4):
        N, nh = self.N, self.nh
        lam = np.empty(N)
        phi = np.empty((N, nh))
        th2 = np.empty(N)
        wH = np.empty(nh)
        th1 = C.c_double()
        it = C.c_int()
        hist = np.zeros(abs(max_it))
        _chk(lib.orc_inner_scf(self._h, dp(f64(lambdas)), tol, max_it, floor, pad, dp(lam), dp(phi), dp(th2), dp(wH),
                               C.byref(th1), C.byref(it), dp(hist), abs(max_it)))
        return dict(lambda_=lam, phi_H=phi, theta2=th2, w_H=wH, theta1=th1.value, iterations=it.value,
                    history=hist[:it.value])

    def expand_last(self):
        orb = np.empty((self.n, self.N))
        w = np.empty(self.n)
        _chk(lib.orc_expand_last(self._h, dp(orb), dp(w)))
        return orb, w

    def f_g(self, phi_H, theta2, w_H, theta1, want_A2=False):
        f = np.empty(self.nh)
        g = C.c_double()
        A2 = np.empty(self.nh * self.nh) if want_A2 else None
        _chk(lib.orc_blocks_f_g(self._h, dp(f64(phi_H)), dp(f64(theta2)), dp(f64(w_H)), theta1, dp(f), C.byref(g),
                                dp(A2)))
        return f, g.value, (A2.reshape(self.nh, self.nh, order="F") if want_A2 else None)


def dorfler_mark(eta, total, theta):
    """est::dorfler_mark (proj/src/estimator.cpp:87-104)"""
    eta = f64(eta)
    out = np.empty(len(eta), np.int32)
    n = C.c_int64()
    _chk(lib.orc_dorfler(dp(eta), len(eta), float(total), float(theta), ip(out), C.byref(n)))
    return out[:n.value].copy()


def keast():
    b = np.empty((11, 4))
    w = np.empty(11)
    _chk(lib.orc_keast(dp(b), dp(w)))
    return b, w


def gen_eig(A, B):
    A = np.asfortranarray(A, np.float64)
    B = np.asfortranarray(B, np.float64)
    n = A.shape[0]
    vals = np.empty(n)
    vecs = np.empty(n * n)
    _chk(lib.orc_gen_eig(n, A.ctypes.data_as(DP), B.ctypes.data_as(DP), dp(vals), dp(vecs)))
    return vals, vecs.reshape(n, n, order="F")


def solve_bordered(A, M, b, beta, c, gamma, nev, floor=1e-8):
    A = np.asfortranarray(A, np.float64)
    M = np.asfortranarray(M, np.float64)
    n = A.shape[0]
    lam, th, sc = C.c_double(), C.c_double(), C.c_double()
    phi = np.empty(n)
    _chk(lib.orc_solve_bordered(n, A.ctypes.data_as(DP), M.ctypes.data_as(DP), dp(f64(b)), beta, dp(f64(c)), gamma,
                                nev, floor, C.byref(lam), dp(phi), C.byref(th), C.byref(sc)))
    return lam.value, phi, th.value, sc.value
