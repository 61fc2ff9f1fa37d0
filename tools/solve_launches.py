"""One C4 capacitance extraction (after warm-up) for an ncu launch list: which kernels fill the solve."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2004_02609_b200 as vc  # noqa: E402
import voxgen  # noqa: E402
st = voxgen.config(sys.argv[1] if len(sys.argv) > 1 else "C4")
ctx = vc.VoxCap(0)
ctx.set_structure(st); ctx.build_operator()
ctx.solve_capacitance(tol=1e-4)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
ctx.solve_capacitance(tol=1e-4)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
