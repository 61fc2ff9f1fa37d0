for cfg in "VC_P2=0 VC_P4=32" "VC_P2=32 VC_P4=32" "VC_P2=64 VC_P4=32"; do
  env $cfg timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/knob.log 2>&1
  echo "$cfg $(tail -1 gpurun_out/knob.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["matvec_ms"],4), [round(x,4) for x in d["pass_ms_mean"]], round(d["ms_per_step"],1))')" >> gpurun_out/knobs.txt
done
VC_P2=32 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "matvec" > gpurun_out/knob_tests.log 2>&1; tail -1 gpurun_out/knob_tests.log >> gpurun_out/knobs.txt
