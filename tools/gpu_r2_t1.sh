set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" 
timeout 1500 python -m pytest tests/test_gpu_reduced.py tests/test_gpu_parity.py -m gpu -x -q -k "reduced or row_sampled or solve_matches or capacitance_c2" 2>&1 | tail -30 > gpurun_out/r2_t1.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_b1.json 2> gpurun_out/r2_b1.err
tail -3 gpurun_out/r2_t1.log; cat gpurun_out/r2_b1.json | head -c 600
