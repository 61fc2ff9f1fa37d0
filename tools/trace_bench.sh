# bench.py under VC_TRACE, per process: ms_per_step and the mean host phase times
for i in 1 2 3 4 5; do
  VC_TRACE=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/tb.json 2> gpurun_out/tb.err
  python - <<'PY'
import json, re, collections
d = json.loads(open("gpurun_out/tb.json").read().strip().splitlines()[-1])
acc = collections.defaultdict(list)
for ln in open("gpurun_out/tb.err"):
    m = re.match(r"\[vc (\S+)\] (.+?)\s+([0-9.]+) ms", ln)
    if m:
        acc[m.group(1) + ":" + m.group(2).strip()].append(float(m.group(3)))
print(round(d["ms_per_step"], 2), {k: round(sum(v) / len(v), 2) for k, v in acc.items() if sum(v) / len(v) > 0.2})
PY
done
