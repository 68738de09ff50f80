timeout 600 python tools/nshapes_probe.py 2>&1 | grep -v "^{" > gpurun_out/r2_nshapes_v3.txt; cat gpurun_out/r2_nshapes_v3.txt
PART=1 bash tools/gpu/final.sh
TAG=s3d bash tools/gpu/bench_all.sh
