set -x; mkdir -p gpurun_out
timeout 900 python tools/nshapes_probe.py > gpurun_out/r2_nshapes.txt 2>&1; cat gpurun_out/r2_nshapes.txt
