set -x; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/r2_pytest_gpu_5.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r2_pytest_gpu_5.log
timeout 300 python tools/pull_profile.py cfg2_mlp5x8192_b512.opt 3 > gpurun_out/r2_pull_steps.txt 2>&1; head -6 gpurun_out/r2_pull_steps.txt
timeout 300 python tools/pull_profile.py cfg2_mlp5x8192_b512.loop 3 > gpurun_out/r2_pull_steps_loop.txt 2>&1; head -8 gpurun_out/r2_pull_steps_loop.txt
