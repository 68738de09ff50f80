set -x; mkdir -p gpurun_out
timeout 900 python tools/overlap_probe.py > gpurun_out/r2_overlap_probe.txt 2>&1; echo "probe exit $?"; cat gpurun_out/r2_overlap_probe.txt
