"""Per-pass device times of the matvec chain on a config (CUDA events via vc_set_timing):
single-column and batched (pair) launches, n repetitions each.  No profiler attached."""
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
ap.add_argument("--n", type=int, default=20)
ap.add_argument("--zmode", type=int, default=0)
ap.add_argument("--tucker", type=int, default=0, help="tucker_digits (0 = exact spectra)")
a = ap.parse_args()
st = voxgen.config(a.config)
ctx = vc.VoxCap(0)
ctx.set_structure(st)
ctx.build_operator(zmode=a.zmode, tucker_digits=a.tucker)
if a.tucker:
    s0 = ctx.stats()
    print(a.config, "tucker", a.tucker, "setup_ms", round(s0["ms_setup"], 2), "resident doubles", s0["spectra_doubles"],
          "err", s0["tucker_err"], "ranks", ctx.tucker()["ranks"])
x = torch.from_numpy(voxgen.seeded_vector(ctx.n, 0)).cuda()
X = torch.stack([x, x.flip(0)], dim=1).contiguous()
for label, fn in (("single", lambda: ctx.matvec(x)), ("pair", lambda: ctx.matvec_batch(X))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ctx.set_timing(True)
    ctx.reset_stats()
    for _ in range(a.n):
        fn()
    torch.cuda.synchronize()
    s = ctx.stats()
    ctx.set_timing(False)
    np_ = max(1, s["n_pass"][0])
    print(a.config, label, "grid", ctx.grid(), "pass_ms",
          [round(s["ms_pass"][i] / max(1, s["n_pass"][i]), 4) for i in range(5)],
          "matvec_ms/launch", round(s["ms_matvec"] / np_, 4),
          "GB/s per pass", [round(s["bytes_moved"][i] / max(1e-9, s["ms_pass"][i] * 1e-3) / 1e9) for i in range(5)])
# preconditioner apply (single column, device vectors) and its stored block size
r = torch.from_numpy(voxgen.seeded_vector(ctx.n, 3)).cuda()
for _ in range(3):
    ctx.precond(r)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(a.n):
    ctx.precond(r)
e1.record()
torch.cuda.synchronize()
print(a.config, "precond apply ms", round(e0.elapsed_time(e1) / a.n, 4), "blocks MB", ctx.stats()["precond_doubles"] * 8 / 1e6)
