import sys, threading, time
sys.path.insert(0, '/root/repo')
import numpy as np, voxgen, paper_2004_02609_b200 as vc
st = voxgen.config("C2")
W = 2
grp = vc.ThreadGroup(W)
ctxs = [vc.VoxCap(0) for _ in range(W)]
out = [None]*W
def work(r):
    try:
        c = ctxs[r]; c.init_distributed(r, W, group=grp); c.set_structure(st); c.build_operator()
        print(r, "built NL", len(c.local_panels()), flush=True)
        z = c.precond(np.ones(len(c.local_panels())))
        print(r, "precond ok", np.isfinite(z).all(), flush=True)
        x, info = c.solve(np.ones(len(c.local_panels())), tol=1e-8, maxit=300)
        print(r, "solve", info, flush=True)
        out[r] = c.solve_capacitance(tol=1e-12, maxit=4000)
        print(r, "cap", out[r][1], flush=True)
    except Exception as e:
        print(r, "ERR", repr(e), flush=True)
th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(W)]
[t.start() for t in th]; [t.join(60) for t in th]
print("alive", [t.is_alive() for t in th], flush=True)
