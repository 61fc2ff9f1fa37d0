# A/B of P3 direct-z variants on C4 pair launches
for ks in 0 1; do for v in 2 3; do VC_P3M_KS=$ks VC_P3M_NST=$v python tools/pass_time.py --config C4 --n 20 2>&1 | grep pair | sed "s/^/ks=$ks nst=$v /"; done; done > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
