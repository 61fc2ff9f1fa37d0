"""Focused driver for ncu: build the operator of a config and run n matvecs (C ABI)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_02609_b200 as vc  # noqa: E402
import voxgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--n", type=int, default=5)
ap.add_argument("--batch", type=int, default=1, help="columns per matvec (vc_matvec_batch)")
ap.add_argument("--tucker", type=int, default=0, help="tucker_digits (0 = exact spectra)")
a = ap.parse_args()
st = voxgen.config(a.config)
ctx = vc.VoxCap(0)
ctx.set_structure(st)
ctx.build_operator(tucker_digits=a.tucker)
x = torch.from_numpy(voxgen.seeded_vector(ctx.n, 0)).cuda()
X = torch.stack([x] * a.batch, dim=1)
for _ in range(a.n):
    y = ctx.matvec(x) if a.batch == 1 else ctx.matvec_batch(X)
torch.cuda.synchronize()
print("ok", a.config, ctx.n, ctx.grid(), float(y.abs().sum()))
