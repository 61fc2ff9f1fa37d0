mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/q_smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/q_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/q_gpu_tests.log
timeout 600 python bench.py > gpurun_out/q_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/q_bench.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/q_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/q_smoke.log
timeout 300 python tools/c5_probe.py > gpurun_out/q_c5.log 2>&1; echo "c5 rc=$?" >> gpurun_out/q_c5.log
