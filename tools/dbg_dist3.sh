timeout 500 python - > gpurun_out/dbg3.log 2>&1 <<'PY'
import faulthandler, sys, threading, traceback
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
faulthandler.dump_traceback_later(400, exit=True)
import test_gpu_distributed as T
for it in range(6):
    for name, W in [("C1", 2), ("R2", 2), ("C2", 2), ("R4", 3)]:
        try:
            T.test_distributed_capacitance(name, W)
            print("ok", it, name, flush=True)
        except Exception as e:
            print("FAIL", it, name, repr(e), flush=True)
            traceback.print_exc()
PY
echo "rc=$?" >> gpurun_out/dbg3.log
