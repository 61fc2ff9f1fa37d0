"""Small invocations of every device path for compute-sanitizer (memcheck / racecheck /
synccheck): panel indexing, both z modes (k_p3 z-FFT, k_p3m direct-z with its mbarrier + TMA
ring), single and batched matvecs, preconditioner, GMRES, capacitance."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2004_02609_b200 as vc  # noqa: E402
import voxgen  # noqa: E402

ctx = vc.VoxCap(0)
for name in ("C1", "C2", "R5"):
    st = voxgen.config(name)
    ctx.set_structure(st)
    for zmode in (1, 2):
        ctx.build_operator(zmode=zmode, box=(4, 4, 4))
        x = voxgen.seeded_vector(ctx.n, 1)
        y = ctx.matvec(x)
        Y = ctx.matvec_batch(np.stack([x, 2 * x], axis=1))
        z = ctx.precond(y)
        C, info = ctx.solve_capacitance(tol=1e-8, maxit=500)
        print(name, zmode, ctx.n, float(np.abs(Y[:, 1] - 2 * y).max()), C.ravel()[:2], [i["iters"] for i in info])
ctx.close()
print("sanitize run done")
