"""cfg2 operator (bench.py's workload) -> a few fixed-count CG iterations; for ncu captures of one SpMM variant
(select with KSB_SPMM_DIA / KSB_DIA_G / KSB_SPMM_T8) and for per-kernel CUDA-event times (--time)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2103_02824_b200 as kb  # noqa: E402

ctx = kb.Context(0)
h = kb.Hierarchy()
h.push(kb.Mesh.box([-bench.BOX] * 3, [bench.BOX] * 3, bench.GRID))
L = kb.Level(ctx, h, 0)
L.assemble(kb.MAT_USER0, c_s=0.5, c_m=0.5, potential=(kb.POT_GAUSSIAN, bench.gaussians()))
dB = ctx.to_device(bench.rhs_block(L.ni))
dX = ctx.empty((L.ni, 16))
its = int(sys.argv[1]) if len(sys.argv) > 1 else 3
L.cg_solve(kb.MAT_USER0, dB, dX, 16, opts=L.cg_options(fixed_iterations=its))
ctx.sync()
if "--time" in sys.argv:
    ctx.set_profiling(True)
    ctx.reset_counters()
    L.cg_solve(kb.MAT_USER0, dB, dX, 16, opts=L.cg_options(fixed_iterations=50))
    ctx.sync()
    for k in ("spmm", "cg_update_r", "cg_update_px"):
        print(k, ctx.kernel_time(k))
