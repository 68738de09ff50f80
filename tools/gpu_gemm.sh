#!/bin/bash
# One gpurun call: GEMM numerics + micro-bench (clocks sampled alongside), then ncu captures.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/gemm_clocks.csv &
SMI=$!
timeout 900 python tools/gemm_check.py --bench > gpurun_out/gemm_check.log 2>&1; echo "gemm_check rc=$?"
kill $SMI
python3 - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/gemm_clocks.csv")))[1:]
mhz = sorted(int(r[1].split()[0]) for r in rows if r and r[1].strip().split()[0].isdigit() and float(r[3].split()[0]) > 300)
print("clocks under load: n=%d median=%s min=%s reasons=%s" % (len(mhz), mhz[len(mhz)//2] if mhz else None, mhz[0] if mhz else None, sorted({r[4].strip() for r in rows if r})))
PY
grep -E "BAD|bench|ALL|knobs" gpurun_out/gemm_check.log
i=0
for cfg in ${NCU_CFGS}; do
  args=$(echo $cfg | tr ':' ' ')
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -s 3 -c 1 -f -o gpurun_out/gemm_prof_$i python tools/gemm_check.py --one $args > gpurun_out/gemm_prof_$i.log 2>&1
  echo "ncu $cfg rc=$?"
  i=$((i+1))
done
