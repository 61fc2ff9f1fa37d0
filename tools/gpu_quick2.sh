timeout 120 python -m pytest tests -m gpu -x -q -k "dense_parity and R1" > gpurun_out/gpu_first.log 2>&1 || { echo "first rc=$?" >> gpurun_out/gpu_first.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python tools/solve_timing.py C4 > gpurun_out/solve_timing.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
