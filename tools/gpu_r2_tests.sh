# round-2 GPU check: full GPU suite + full-size parity (logs and JSON under gpurun_out/)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t_build.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q --timeout 1200 > gpurun_out/t_fullsize.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu --timeout 900 --deselect tests/test_gpu_fullsize.py > gpurun_out/t_gpu.log 2>&1
tail -n 3 gpurun_out/t_fullsize.log gpurun_out/t_gpu.log
