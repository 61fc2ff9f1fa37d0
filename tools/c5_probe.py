"""C5 (2048 x 2048 x 128 crossing bus) on one GPU: geometry, build, one matvec, memory."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2004_02609_b200 as vc, voxgen
t0 = time.time(); st = voxgen.config("C5"); print("voxgen", round(time.time() - t0, 1), "s", st.dims, flush=True)
ctx = vc.VoxCap(0)
lab = torch.from_numpy(st.label).cuda(); eps = torch.from_numpy(st.eps).cuda(); torch.cuda.synchronize()
t0 = time.time(); ctx.set_geometry(lab, eps, st.eps_out, st.dv); torch.cuda.synchronize()
print("N", ctx.n, "Nc", ctx.n_cond, "m", ctx.m, "set_geometry", round(time.time() - t0, 2), "s", flush=True)
del lab, eps; torch.cuda.empty_cache()
t0 = time.time(); ctx.build_operator(); torch.cuda.synchronize()
s = ctx.stats(); print("grid", ctx.grid(), "build", round(time.time() - t0, 2), "s", {k: round(s[k], 1) for k in ("ms_kgen", "ms_kfft", "ms_precond_build")}, flush=True)
free, total = torch.cuda.mem_get_info(); print("device memory used GB", round((total - free) / 2**30, 1), flush=True)
x = torch.from_numpy(voxgen.seeded_vector(ctx.n, 0)).cuda()
ctx.set_timing(True)
for i in range(3):
    ctx.reset_stats(); y = ctx.matvec(x); torch.cuda.synchronize()
    s = ctx.stats()
    print("matvec ms", round(s["ms_matvec"], 2), "passes", [round(v, 2) for v in s["ms_pass"]], "GB", round(s["bytes_matvec"] / 1e9, 1), flush=True)
np.save("gpurun_out/c5_y_rows.npy", y.cpu().numpy()[:: max(1, ctx.n // 4096)])
