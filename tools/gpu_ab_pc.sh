for v in 0 1; do VC_PC_ROWWARP=$v python tools/pass_time.py --config C4 --n 20 2>&1 | tail -1 | sed "s/^/rowwarp=$v /"; done
