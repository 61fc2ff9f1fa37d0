# one iteration: GPU tests (subset regex $1, "all" = everything), bench, optional ncu of kernel $2
SEL=${1:-all}; KR=${2:-}; TAG=${3:-it}
python -c "import __graft_entry__ as g; g.build()" > /dev/null
if [ "$SEL" = "all" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/${TAG}_tests.log
elif [ "$SEL" != "none" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$SEL" 2>&1 | tail -15 > gpurun_out/${TAG}_tests.log
fi
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python - <<PY
import json
d=json.load(open("gpurun_out/${TAG}_bench.json"))
print("step_ms", round(d["ms_per_step"],2), "value %.3e"%d["value"], "e2e %.3e"%d["e2e"]["value"], "matvec_ms", round(d["matvec_ms"],4))
print("pass_ms", [round(x,4) for x in d["pass_ms_mean"]], "pass_gbs", [round(x) for x in d["pass_gbs"]])
print("roofline", d["roofline"])
PY
if [ -n "$KR" ]; then bash tools/gpu_prof2.sh $KR C4 2 ${TAG}_prof; fi
tail -3 gpurun_out/${TAG}_tests.log 2>/dev/null
