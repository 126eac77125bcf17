"""ctypes binding of libksb.so (the C-ABI declared in include/ksb.h).

The product path has no CPU fallback: if the in-tree library is missing this
module raises at import time, and every compute entry point runs on the GPU.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_lib" / "libksb.so"

if not LIB_PATH.exists():
    raise ImportError(
        f"libksb.so not found at {LIB_PATH}; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        " (there is no CPU fallback for the product path)")

lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_GLOBAL if hasattr(os, "RTLD_GLOBAL") else 0)

P = C.c_void_p
PP = C.POINTER(C.c_void_p)
I = C.c_int
I64 = C.c_int64
D = C.c_double
DP = C.POINTER(C.c_double)
IP = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)
CP = C.c_char_p


class CgOpts(C.Structure):
    _fields_ = [("tol", D), ("max_iterations", I), ("fixed_iterations", I), ("precond", I), ("check_every", I)]


class CgStats(C.Structure):
    _fields_ = [("iterations", I), ("relative_residual", D), ("converged", I), ("breakdown", I)]


class StepOpts(C.Structure):
    _fields_ = [("tol_linear", D), ("tol_inner", D), ("score_floor", D), ("max_inner", I), ("nev_pad", I),
                ("check_every", I), ("fixed_sweeps", I), ("norm_l1", I),
                ("precond", I)]


class ScfOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iterations", C.c_int), ("mixing", C.c_double), ("hartree_on", C.c_int),
                ("xc_on", C.c_int), ("tol_eig", C.c_double), ("norm_l1", C.c_int)]


class StepLog(C.Structure):
    _fields_ = [("inner_iterations", I), ("hartree_iterations", I), ("delta", D), ("ms_bvp", D), ("ms_hartree", D),
                ("ms_project", D), ("ms_inner", D), ("ms_total", D), ("cg_iterations", I64)]


SOP = C.POINTER(StepOpts)
SLP = C.POINTER(StepLog)

# name -> (restype, argtypes); mirrors include/ksb.h exactly (checked by tests/test_abi.py)
PROTOTYPES = {
    "ksb_last_error": (CP, []),
    "ksb_code_name": (CP, [I]),
    "ksb_version": (I, []),
    "ksb_mesh_box": (I, [DP, DP, I, PP]),
    "ksb_mesh_uniform_refine": (I, [P, PP]),
    "ksb_mesh_adapt_refine": (I, [P, IP, I64, PP]),
    "ksb_mesh_free": (None, [P]),
    "ksb_mesh_sizes": (I, [P, I64P]),
    "ksb_mesh_get": (I, [P, I, P]),
    "ksb_hier_create": (I, [PP]),
    "ksb_hier_push": (I, [P, P]),
    "ksb_hier_mesh": (I, [P, I, PP]),
    "ksb_hier_save": (I, [P, C.c_char_p]),
    "ksb_hier_load": (I, [C.c_char_p, PP]),
    "ksb_mesh_save": (I, [P, C.c_char_p]),
    "ksb_mesh_load": (I, [C.c_char_p, PP]),
    "ksb_state_save": (I, [C.c_char_p, I, I, C.c_int64, C.c_int64, DP, DP, I, DP]),
    "ksb_state_sizes": (I, [C.c_char_p, P]),
    "ksb_state_load": (I, [C.c_char_p, DP, DP, I, DP]),
    "ksb_hier_free": (None, [P]),
    "ksb_hier_levels": (I, [P]),
    "ksb_hier_prolongation": (I, [P, I, IP, DP]),
    "ksb_ctx_create": (I, [I, PP]),
    "ksb_ctx_destroy": (None, [P]),
    "ksb_ctx_stream": (I, [P, PP]),
    "ksb_ctx_sync": (I, [P]),
    "ksb_ctx_set_profiling": (I, [P, I]),
    "ksb_ctx_kernel_time": (I, [P, CP, DP, I64P]),
    "ksb_ctx_kernel_launches": (I, [P, I64P]),
    "ksb_ctx_reset_counters": (I, [P]),
    "ksb_malloc": (I, [P, PP, I64]),
    "ksb_free": (I, [P, P]),
    "ksb_memcpy_h2d": (I, [P, P, P, I64]),
    "ksb_memcpy_d2h": (I, [P, P, P, I64]),
    "ksb_level_create": (I, [P, P, I, PP]),
    "ksb_level_destroy": (None, [P]),
    "ksb_level_sizes": (I, [P, I64P]),
    "ksb_level_index": (I, [P, I, P]),
    "ksb_mat_assemble": (I, [P, I, D, D, I, I, DP, D, P, D]),
    "ksb_mat_axpby": (I, [P, I, D, I, D, I]),
    "ksb_mat_values": (I, [P, I, I, DP]),
    "ksb_spmm": (I, [P, I, P, I, I, P, I]),
    "ksb_cg_defaults": (I, [C.POINTER(CgOpts)]),
    "ksb_cg_solve": (I, [P, I, I, DP, P, P, I, I, C.POINTER(CgOpts), C.POINTER(CgStats)]),
    "ksb_cg_solve_host": (I, [P, I, I, DP, P, P, I, I, C.POINTER(CgOpts), C.POINTER(CgStats)]),
    "ksb_solve": (I, [P, I, P, P, C.POINTER(CgOpts), P, C.POINTER(CgStats)]),
    "ksb_mat_min_diag": (I, [P, I, DP]),
    "ksb_step_defaults": (I, [SOP]),
    "ksb_scf_defaults": (I, [C.POINTER(ScfOpts)]),
    "ksb_coarse_scf": (I, [P, C.POINTER(ScfOpts), DP, P, I, P, P, IP, DP, I]),
    "ksb_system_set": (I, [P, DP, I, I, D, I, D, D, I, I]),
    "ksb_level_ops": (I, [P]),
    "ksb_correction_step": (I, [P, SOP, DP, P, I, P, SLP, IP, IP]),
    "ksb_mlc_begin": (I, [P, SOP, DP, P, I, P, SLP, IP, IP]),
    "ksb_mlc_sweep": (I, [P, SOP, DP, P, I, DP]),
    "ksb_mlc_finish": (I, [P, SOP, P, P]),
    "ksb_correction_step_host": (I, [P, SOP, DP, P, I, P, SLP, IP, IP]),
    "ksb_density_xc": (I, [P, P, I, I, P, P]),
    "ksb_moments": (I, [P, P, DP]),
    "ksb_boundary_values": (I, [P, DP, P]),
    "ksb_sqload": (I, [P, P, I, I, P]),
    "ksb_hartree_solve": (I, [P, P, I, I, P, D, P, IP]),
    "ksb_outer_solve": (I, [P, SOP, P, P, DP, P, I, P, IP, IP, DP]),
    "ksb_sqload_full": (I, [P, P, I, I, D, P]),
    "ksb_density": (I, [P, P, I, I, D, P]),
    "ksb_xc_field": (I, [P, I, D, D, P, P]),
    "ksb_indicators": (I, [P, DP, P, I, P, P, P, DP]),
    "ksb_prolong": (I, [P, P, I, I, I, P, I, I]),
    "ksb_dorfler_mark": (I, [DP, C.c_int64, D, D, IP, C.POINTER(C.c_int64)]),
    "ksb_outer_build": (I, [P, I, P, P, DP]),
    "ksb_outer_apply": (I, [P, SOP, DP, P, I, I, P, IP, IP]),
    "ksb_prepare_blocks": (I, [P, P, I, P, P, P]),
    "ksb_blocks_get": (I, [P, I, DP]),
    "ksb_inner_scf": (I, [P, SOP, DP, DP, DP, DP, DP, DP, IP, DP, I]),
    "ksb_expand": (I, [P, P, I, P, P, P, P]),
    "ksb_norms": (I, [P, P, DP]),
    "ksb_l1_norm": (I, [P, P, DP]),
    "ksb_energy": (I, [P, P, I, I, P, DP]),
}

for _name, (_res, _args) in PROTOTYPES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

CODE_NAMES = {0: "ok", 1: "nonconvergence", 2: "mismatched-spaces", 3: "singular-quadrature",
              4: "ambiguous-selection", 5: "internal", 6: "invalid-argument", 7: "invalid-domain",
              8: "hierarchy", 9: "io", 10: "cuda"}


class KsbError(RuntimeError):
    """Mirror of ksafem::Error: `code` is the reference's machine code string."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.code = CODE_NAMES.get(status, "unknown")
        super().__init__(message)


def check(status: int) -> None:
    if status != 0:
        raise KsbError(status, lib.ksb_last_error().decode())
