# round profile set: launch list of the bench command + ncu --set full of the dominant kernels
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
timeout 200 python tools/prof_matvec.py --config C4 --n 3 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p[1-5]" -s 5 -c 5 -o gpurun_out/prof_c4 python tools/prof_matvec.py --config C4 --n 3 > gpurun_out/ncu2.log 2>&1
timeout 200 python tools/prof_matvec.py --config C3 --n 3 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p[1-5]" -s 5 -c 5 -o gpurun_out/prof_c3 python tools/prof_matvec.py --config C3 --n 3 > gpurun_out/ncu3.log 2>&1
echo done
