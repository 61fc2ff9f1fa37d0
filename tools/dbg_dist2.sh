timeout 400 python - > gpurun_out/dbg2.log 2>&1 <<'PY'
import faulthandler, sys, threading
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
faulthandler.dump_traceback_later(150, exit=True)
import test_gpu_distributed as T
for name, W in [("C1", 2), ("R2", 2), ("C2", 2)]:
    print("running", name, W, flush=True)
    T.test_distributed_capacitance(name, W)
    print("ok", name, flush=True)
PY
echo "rc=$?" >> gpurun_out/dbg2.log
