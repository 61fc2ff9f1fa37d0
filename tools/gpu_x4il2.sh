# compile-time X4 layout flag in P5: C4 / C3 pass times, C5 probe, C5 + parity tests first, bench, then the rest of the suite
mkdir -p gpurun_out
timeout 200 python tools/pass_time.py --config C4 --n 20 > gpurun_out/pass_times_v18.txt 2>&1
timeout 200 python tools/pass_time.py --config C3 --n 20 >> gpurun_out/pass_times_v18.txt 2>&1
timeout 600 python tools/c5_probe.py > gpurun_out/c5_single_gpu_v18.txt 2>&1; echo "c5 rc=$?" >> gpurun_out/c5_single_gpu_v18.txt
timeout 300 python bench.py > gpurun_out/bench_v18.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_v18.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v18.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_v18.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_v18.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_v18.log
cat gpurun_out/pass_times_v18.txt; tail -4 gpurun_out/c5_single_gpu_v18.txt; tail -3 gpurun_out/gpu_tests_v18.log
