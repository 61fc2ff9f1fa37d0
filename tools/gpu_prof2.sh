# ncu --set full of one kernel (regex $1) on config $2, batch $3, via tools/prof_matvec.py
KR=${1:-k_p3m}; CF=${2:-C4}; NB=${3:-2}; OUT=${4:-prof}
timeout 200 python tools/prof_matvec.py --config $CF --n 3 --batch $NB > gpurun_out/plain_prof.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KR -s 1 -c ${NC:-1} -o gpurun_out/$OUT python tools/prof_matvec.py --config $CF --n 3 --batch $NB > gpurun_out/ncu_prof.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_prof.log
