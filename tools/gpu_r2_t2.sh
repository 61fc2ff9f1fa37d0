# P3 DMMA kernel: full GPU suite, then bench and the P3 capture
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r2_t2_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_t2_bench.json 2> gpurun_out/r2_t2_bench.err
tail -5 gpurun_out/r2_t2_tests.log; head -c 1500 gpurun_out/r2_t2_bench.json
