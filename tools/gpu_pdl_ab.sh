# A/B of programmatic dependent launch on the matvec passes (VOXCAP_PDL=0 plain launches), then the
# GPU suite with the default (PDL on), then the follow-up evidence of tools/gpu_final.sh
mkdir -p gpurun_out
for r in 1 2; do for v in 0 1; do
  VOXCAP_PDL=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_pdl${v}_r$r.log 2>&1
  echo "pdl=$v run=$r rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_pdl${v}_r$r.log) $(grep -o '"solve_s_per_column": [0-9.]*' gpurun_out/ab_pdl${v}_r$r.log)" >> gpurun_out/ab_pdl.txt
done; done
for v in 0 1; do VOXCAP_PDL=$v timeout 300 python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_pdl${v}_c3.log 2>&1
  echo "C3 pdl=$v rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_pdl${v}_c3.log)" >> gpurun_out/ab_pdl.txt; done
cat gpurun_out/ab_pdl.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_pdl.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_pdl.log
tail -3 gpurun_out/gpu_tests_pdl.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_pdl.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_pdl.log
timeout 300 python bench.py > gpurun_out/bench_pdl.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_pdl.log
bash tools/gpu_final.sh
