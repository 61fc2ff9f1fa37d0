# C5 one-GPU P4 half-sector fix (X4 interleaved when P4's tile is one kx wide): C5 probe, C4 / C3 pass
# times (unchanged layouts there), then the GPU suite, smoke and the default bench line
mkdir -p gpurun_out
timeout 600 python tools/c5_probe.py > gpurun_out/c5_single_gpu_x4il.txt 2>&1; echo "c5 rc=$?" >> gpurun_out/c5_single_gpu_x4il.txt
tail -5 gpurun_out/c5_single_gpu_x4il.txt
timeout 200 python tools/pass_time.py --config C4 --n 20 > gpurun_out/pass_times_x4il.txt 2>&1
timeout 200 python tools/pass_time.py --config C3 --n 20 >> gpurun_out/pass_times_x4il.txt 2>&1
cat gpurun_out/pass_times_x4il.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_x4il.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_x4il.log
tail -3 gpurun_out/gpu_tests_x4il.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_x4il.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_x4il.log
timeout 300 python bench.py > gpurun_out/bench_x4il.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_x4il.log
