# follow-up evidence of the final build: C5 on one GPU (timed matvec passes) and the ncu --set full
# capture of the five passes on C3 (z-FFT mode), summarised on the box
mkdir -p gpurun_out
timeout 600 python tools/c5_probe.py > gpurun_out/c5_single_gpu.txt 2>&1; echo "c5 rc=$?" >> gpurun_out/c5_single_gpu.txt
timeout 200 python tools/prof_matvec.py --config C3 --n 3 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p[1-5]" -s 5 -c 5 -o /tmp/prof_c3 python tools/prof_matvec.py --config C3 --n 3 > gpurun_out/ncu3.log 2>&1
python tools/ncu_summary.py report /tmp/prof_c3.ncu-rep > gpurun_out/c3_passes_full.txt 2>&1
python tools/ncu_stalls.py /tmp/prof_c3.ncu-rep k_p3 > gpurun_out/c3_p3_stalls.txt 2>&1
python tools/ncu_lines.py /tmp/prof_c3.ncu-rep k_p3 20 > gpurun_out/c3_p3_lines.txt 2>&1
echo done; ls -la gpurun_out | tail -8
