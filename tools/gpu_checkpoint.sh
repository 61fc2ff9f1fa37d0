# round checkpoint: GPU tests, smoke, bench line, launch list, full capture of the P3 pair launch
TAG=${1:-r02_ck}
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/${TAG}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
bash tools/gpu_prof2.sh k_p3m C4 2 ${TAG}_p3m
NC=4 bash tools/gpu_prof2.sh "k_p1|k_p2|k_p4s|k_p5" C4 2 ${TAG}_passes
tail -2 gpurun_out/${TAG}_gpu_tests.log; tail -1 gpurun_out/${TAG}_smoke.log; head -c 400 gpurun_out/${TAG}_bench.json
