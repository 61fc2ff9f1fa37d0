# ncu --set full of one kernel (K, default k_p5) on a C4 pair matvec: summary, stalls, top lines
K=${K:-k_p5}; CFG=${CFG:-C4}
mkdir -p gpurun_out
timeout 200 python tools/prof_matvec.py --config $CFG --n 3 --batch 2 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -f -o /tmp/prof_k_$K python tools/prof_matvec.py --config $CFG --n 3 --batch 2 > gpurun_out/ncu2.log 2>&1
python tools/ncu_summary.py report /tmp/prof_k_$K.ncu-rep > gpurun_out/${K}_full.txt 2>&1
python tools/ncu_stalls.py /tmp/prof_k_$K.ncu-rep $K > gpurun_out/${K}_stalls.txt 2>&1
python tools/ncu_lines.py /tmp/prof_k_$K.ncu-rep $K 40 > gpurun_out/${K}_lines.txt 2>&1
cat gpurun_out/${K}_full.txt gpurun_out/${K}_stalls.txt gpurun_out/${K}_lines.txt
