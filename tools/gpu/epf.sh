mkdir -p gpurun_out
timeout 300 python tools/gemm_check.py > gpurun_out/epf_check.txt 2>&1; echo "check $?"; grep -c "^ok" gpurun_out/epf_check.txt; grep BAD gpurun_out/epf_check.txt | head
timeout 600 python tools/epi_sweep.py base nopf=26:0 base2 > gpurun_out/epf_sweep.txt 2>&1; echo "sweep $?"
cat gpurun_out/epf_sweep.txt
timeout 300 python tools/gemm_trace.py 512,8192,8192,0,0,1 512,8192,8192,0,1,2 8192,8192,512,1,0,3:6 > gpurun_out/epf_trace.txt 2>&1; cat gpurun_out/epf_trace.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/epf_pytest.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/epf_pytest.log
timeout 600 python bench.py --no-variants --no-cpu-baseline > gpurun_out/epf_bench.json 2>/dev/null; echo "bench $?"; cut -c1-250 gpurun_out/epf_bench.json
