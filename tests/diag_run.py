import sys, json, time
sys.path.insert(0, '/root/repo')
import paper_2103_02824_b200 as kb
from paper_2103_02824_b200.driver import run
ctx = kb.Context(0)
for refine, levels in [("uniform", 4), ("adaptive", 5)]:
    t = time.time()
    log = run(ctx, [[2.0, 0, 0, 0]], 1, 2.0, "lda", 10.0, 8, levels, refine=refine)
    print(refine, "aborted", log.aborted, log.abort_reason[:120], "wall", round(log.wall_seconds, 3))
    for r in log.records:
        print(" ", r.level, r.n_dofs, r.lambdas, round(r.energy[4], 8), r.eta_sq_total, r.outer_iterations, round(r.t_total, 3))
