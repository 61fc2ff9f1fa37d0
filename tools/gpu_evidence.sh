# round evidence: GPU suite, default bench line, launch list of the bench command, ncu --set full
# of the matvec passes on C4 (batched column pair) and C3, summarised on the box
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
python tools/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
gzip -f gpurun_out/launches.csv
timeout 200 python tools/prof_matvec.py --config C4 --n 3 --batch 2 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p[1-5]" -s 5 -c 5 -o /tmp/prof_c4b python tools/prof_matvec.py --config C4 --n 3 --batch 2 > gpurun_out/ncu2.log 2>&1
python tools/ncu_summary.py report /tmp/prof_c4b.ncu-rep > gpurun_out/passes_full.txt 2>&1
python tools/ncu_stalls.py /tmp/prof_c4b.ncu-rep k_p3m > gpurun_out/p3_stalls.txt 2>&1
timeout 200 python tools/pass_time.py --config C4 --n 20 > gpurun_out/pass_times.txt 2>&1
timeout 200 python tools/pass_time.py --config C3 --n 20 >> gpurun_out/pass_times.txt 2>&1
timeout 300 python bench.py --config C3 --steps 5 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
timeout 300 python bench.py --tucker 10 --steps 5 --no-cpu-baseline > gpurun_out/bench_tucker.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
echo done
python tools/ncu_lines.py /tmp/prof_c4b.ncu-rep k_p3m 20 > gpurun_out/p3_lines.txt 2>&1; ls -la gpurun_out; du -sh gpurun_out
