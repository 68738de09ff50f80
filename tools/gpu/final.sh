# Round-end evidence, in two gpurun calls (one ncu run per call):
#   PART=1: GPU tests, smoke, default bench, the bench's ncu launch list
#   PART=2: a full ncu capture of one cfg2 step's GEMMs (profiles/traffic.json)
set -x; mkdir -p gpurun_out/tmp
if [ "${PART:-1}" = 1 ]; then
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2_final_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2_final_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_final_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/r2_final_smoke.log
timeout 900 python bench.py > gpurun_out/r2_final_bench.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/r2_final_bench.log | cut -c1-300
timeout 300 python bench.py --steps 2 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/r2_final_bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_final_launches.csv python bench.py --steps 2 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/r2_final_bench_under_ncu.log 2>&1; echo "ncu launches exit $?"
python tools/ncu_summary.py gpurun_out/r2_final_launches.csv > gpurun_out/r2_final_launches_summary.txt 2>&1; head -20 gpurun_out/r2_final_launches_summary.txt
gzip -f gpurun_out/r2_final_launches.csv
else
timeout 300 python tools/ncu_step.py cfg2_mlp5x8192_b512 3 > gpurun_out/r2_final_ncu_step_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:gemm -s 30 -c 15 -f -o gpurun_out/tmp/step python tools/ncu_step.py cfg2_mlp5x8192_b512 3 > gpurun_out/r2_final_ncu_step.log 2>&1; echo "ncu step exit $?"
python tools/ncu_summary.py gpurun_out/tmp/step.ncu-rep > gpurun_out/r2_final_ncu_step_summary.txt 2>&1
python tools/traffic_json.py gpurun_out/tmp/step.ncu-rep fwd,fwd,fwd,fwd,fwd,bwd_w,bwd_x,bwd_w,bwd_x,bwd_w,bwd_x,bwd_w,bwd_x,bwd_w,bwd_x > gpurun_out/r2_final_traffic.json 2>&1; cat gpurun_out/r2_final_traffic.json
fi
rm -rf gpurun_out/tmp
