#!/bin/bash
# One GEMM shape under several debug-knob settings (timed, no profiler):
#   SHAPE="3456 115200 384 1 0 -" KNOBS="base 5:2 6:1 4:3" bash tools/knob_matrix.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for kn in ${KNOBS}; do
  k=$kn; [ "$kn" = base ] && k=""
  echo -n "knobs=$kn  "
  TPX_GEMM_KNOBS="$k" timeout 120 python tools/gemm_check.py --one ${SHAPE} 2>&1 | grep one
done
