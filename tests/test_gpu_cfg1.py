"""cfg1 (BASELINE.json configs[0]) end to end on the device against the oracle's own trajectory.

He (Z=2), one doubly occupied orbital, LDA, [-10,10]^3, 8^3 Kuhn coarse mesh, 3 uniform refinements:
the corrected level loop (proj/src/driver.cpp:94-163) from the oracle's coarse SCF. The oracle's
trajectory is committed in tests/golden/cfg1_oracle_trajectory.json (tests/cfg1_oracle.py made it;
it takes minutes on the CPU). Levels 1 and 2 converge; on level 3 the reference algorithm itself
stalls in a two-cycle of the inner iteration at outer step 4, and the device path must reproduce that
failure (same step, same error text) after the same four steps.
"""
import json
from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden" / "cfg1_oracle_trajectory.json"
FINAL = Path(__file__).resolve().parent / "golden" / "cfg1_oracle_final.npz"  # converged levels 1, 2


def test_cfg1_golden_is_self_consistent():
    g = json.loads(GOLDEN.read_text())["levels"]
    assert [lv["level"] for lv in g] == [1, 2, 3]
    assert g[0]["steps"][-1]["delta"] < 1e-6 and g[1]["steps"][-1]["delta"] < 1e-6
    assert "error" in g[2]["steps"][-1]


@pytest.mark.gpu
def test_cfg1_trajectory_matches_oracle():
    from cfg1_parity import run

    g = json.loads(GOLDEN.read_text())["levels"]
    out = run(levels=3, oracle_levels=0, verbose=False)
    gpu = out["gpu"]
    assert len(gpu) == 2
    for rec, ref in zip(gpu, g[:2]):
        steps = ref["steps"]
        assert rec["outer"] == len(steps)
        assert rec["inner"] == [s["inner"] for s in steps]
        lam = np.array([s["lambda"][0] for s in steps])
        glam = np.array([x[0] for x in rec["lambdas"]])
        assert np.max(np.abs(glam - lam) / np.abs(lam)) < 1e-8
        d, gd = np.array([s["delta"] for s in steps]), np.array(rec["deltas"])
        # delta is an H1 norm of a density difference: absolute floor at the linear-solve tolerance
        assert np.all(np.abs(gd - d) <= 1e-6 * d + 1e-9)
        e, ge = np.array(ref["energy"]), np.array(rec["energy"])
        assert np.max(np.abs(ge - e) / np.abs(e)) < 1e-8  # total energy and its parts, 1e-8 relative
    ref = np.load(FINAL)
    for lev in (1, 2):
        fo, fw = ref[f"orb_level{lev}"][:, 0], ref[f"w_level{lev}"]
        go, gw = out["finals"][lev]["orb"][:, 0], out["finals"][lev]["w"]
        go = go * np.sign(go @ fo)  # sign alignment
        assert np.linalg.norm(go - fo) <= 1e-6 * np.linalg.norm(fo)  # orbital, relative L2
        assert np.linalg.norm(2 * go**2 - 2 * fo**2) <= 1e-6 * np.linalg.norm(2 * fo**2)  # density
        assert np.linalg.norm(gw - fw) <= 1e-6 * np.linalg.norm(fw)  # Hartree potential
    err = out["gpu_error"]
    ref3 = g[2]["steps"]
    assert err["failed_step"] == len(ref3) - 1
    assert err["error"] == ref3[-1]["error"]
    assert err["inner"] == [s["inner"] for s in ref3[:-1]]
    lam = np.array([s["lambda"][0] for s in ref3[:-1]])
    glam = np.array([x[0] for x in err["lambdas"]])
    assert np.max(np.abs(glam - lam) / np.abs(lam)) < 1e-8
