set -x; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q --timeout 600 > gpurun_out/r2_pytest_parity.log 2>&1; echo "parity exit $?"; tail -3 gpurun_out/r2_pytest_parity.log
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/r2_sanitizer_$tool.log 2>&1; echo "$tool exit $?"; tail -12 gpurun_out/r2_sanitizer_$tool.log
done
