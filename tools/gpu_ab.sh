# A/B check of a kernel change: matvec parity subset, a short bench line, and (optional)
# ncu counters of the matvec passes.  usage: gpurun -- 'bash tools/gpu_ab.sh [pytest -k expr]'
K=${1:-"matvec or fft or zmodes"}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$K" > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
tail -3 gpurun_out/ab_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ab_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/ab_bench.log
python - <<'EOF'
import json
for l in open("gpurun_out/ab_bench.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("matvec_ms", round(d["matvec_ms"], 4), "passes", [round(x, 4) for x in d["pass_ms_mean"]],
              "step_ms", round(d["ms_per_step"], 2), "value", "%.4g" % d["value"], "setup", d.get("setup_breakdown_ms"))
EOF
if [ -n "$NCU" ]; then
  timeout 600 ncu --clock-control none -k "regex:$NCU" -s 5 -c 5 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum \
    python tools/prof_matvec.py --config ${CFG:-C4} --n 3 > gpurun_out/ab_ncu.log 2>&1
  grep -E "k_p|gpu__time|dram__bytes|issue_active|bank_conf|warps_active|fp64|wavefronts" gpurun_out/ab_ncu.log | head -80
fi
