#!/bin/bash
# ncu captures of one GEMM shape under several gemm.cu debug-knob settings:
#   SHAPE="8192 8192 512 1 0 3,6" KNOBS="base 7:4 8:1" bash tools/gpu_ncu_knobs.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for kn in ${KNOBS}; do
  k=$kn; [ "$kn" = base ] && k=""
  TPX_GEMM_KNOBS="$k" timeout 600 ncu --set full --clock-control none -k regex:gemm -s 3 -c 1 -f -o gpurun_out/knob_${kn//[:,]/_} python tools/gemm_check.py --one ${SHAPE} > gpurun_out/knob_${kn//[:,]/_}.log 2>&1
  echo "ncu knobs=$kn rc=$?"
done
