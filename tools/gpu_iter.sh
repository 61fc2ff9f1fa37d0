# one iteration: matvec / capacitance parity, then pass times (C4, C3)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reduced.py tests/test_gpu_distributed.py -m gpu -x -q > gpurun_out/iter_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/iter_tests.log
timeout 200 python tools/pass_time.py --config C4 --n 20 > gpurun_out/iter_pass.txt 2>&1
timeout 200 python tools/pass_time.py --config C3 --n 20 >> gpurun_out/iter_pass.txt 2>&1
tail -3 gpurun_out/iter_tests.log; cat gpurun_out/iter_pass.txt
