"""Where does a GMRES solve spend its time?  Device time of matvecs vs the whole solve."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2004_02609_b200 as vc, voxgen
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
st = voxgen.config(cfg)
ctx = vc.VoxCap(0)
ctx.set_structure(st); ctx.build_operator()
for rep in range(6):
    ctx.set_timing(rep % 2 == 1); ctx.reset_stats()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    C, info = ctx.solve_capacitance(tol=1e-4)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    s = ctx.stats()
    print(f"rep {rep} timing={rep%2==1} wall {1e3*(t1-t0):.1f} ms, matvecs {s['n_matvec']}, "
          f"matvec dev {s['ms_matvec']:.1f} ms, launches {s['gpu_launches']}, iters {[i['iters'] for i in info]}")
for rep in range(3):
    t0 = time.perf_counter(); ctx.set_structure(st); t1 = time.perf_counter(); ctx.build_operator(); t2 = time.perf_counter()
    print(f"set_geometry {1e3*(t1-t0):.1f} ms build {1e3*(t2-t1):.1f} ms  stats setup {ctx.stats()['ms_setup']:.1f} geom {ctx.stats()['ms_geometry']:.1f}")
