mkdir -p gpurun_out
timeout 300 python tools/gemm_check.py > gpurun_out/mn4d_check.txt 2>&1; echo "check $?"; grep -c "^ok" gpurun_out/mn4d_check.txt; grep BAD gpurun_out/mn4d_check.txt | head
export SHAPES="fwd,bwd_x,bwd_w"
timeout 600 python tools/epi_sweep.py base old=25:0 > gpurun_out/mn4d_sweep.txt 2>&1; echo "sweep $?"
for l in "8192 8192 512"; do timeout 200 python tools/gemm_layouts.py $l; done >> gpurun_out/mn4d_sweep.txt 2>&1
timeout 200 python tools/gemm_layouts.py 512 8192 8192 >> gpurun_out/mn4d_sweep.txt 2>&1
cat gpurun_out/mn4d_sweep.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/mn4d_pytest.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/mn4d_pytest.log
