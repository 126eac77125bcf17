"""Level driver around the device correction step.

solve_level_corrected mirrors the reference's outer loop (proj/src/driver.cpp:94-163): one
correction step per outer iteration until the H1 norm of the density change drops below
tol_outer, with the same iteration cap and error. prolong() is the nested-space transfer of the
warm start (proj/src/driver.cpp:367-371, fem::SpaceHierarchy::prolong, proj/src/fespace.cpp:76-84).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import api
from ._native import KsbError


def prolong(fine: api.Mesh, coarse_values: np.ndarray) -> np.ndarray:
    """Values on the previous level -> this level: inherited vertices keep theirs, new vertices
    average their parent edge. Parents may themselves be new (bisection chains), so the
    averaging runs in dependency rounds."""
    vp = fine.array("vparent")
    npv = fine.sizes()[5]
    x = np.asarray(coarse_values, np.float64)
    n = fine.n_vertices
    out = np.zeros((n,) + x.shape[1:])
    out[:npv] = x[:npv]
    known = np.zeros(n, bool)
    known[:npv] = True
    todo = np.arange(npv, n)
    while todo.size:
        a, b = vp[todo, 0], vp[todo, 1]
        ready = known[a] & known[b]
        if not ready.any():
            raise RuntimeError("prolongation parents form a cycle")
        v = todo[ready]
        out[v] = 0.5 * out[a[ready]] + 0.5 * out[b[ready]]
        known[v] = True
        todo = todo[~ready]
    return out


@dataclass
class LevelResult:
    level: int
    n_dofs: int
    outer_iterations: int
    lambdas: np.ndarray
    inner_iterations: list = field(default_factory=list)
    deltas: list = field(default_factory=list)
    logs: list = field(default_factory=list)


def solve_level_corrected(L: api.Level, lambdas: np.ndarray, Phi: api.DeviceArray, w: api.DeviceArray,
                          tol_outer: float = 1e-6, max_outer: int = 40, level: int = 0, **step_opts) -> LevelResult:
    """Outer iterations on one level (proj/src/driver.cpp:106-155); state updated in place."""
    res = LevelResult(level=level, n_dofs=L.n, outer_iterations=0, lambdas=lambdas)
    for outer in range(max_outer):
        try:
            lg = L.correction_step(lambdas, Phi, w, **step_opts)
        except KsbError as e:  # keep the trajectory so far for diagnostics, re-raise unchanged
            e.partial = res
            e.step = outer
            raise
        lg["lambda"] = np.array(lambdas, copy=True).tolist()
        res.inner_iterations.append(lg["inner_iterations"])
        res.deltas.append(lg["delta"])
        res.logs.append(lg)
        res.outer_iterations = outer + 1
        if lg["delta"] < tol_outer:
            return res
    raise KsbError(1, f"nonconvergence: outer iteration cap reached on level {level}")
