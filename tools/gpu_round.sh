#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list + full capture of the GEMMs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
STAGES=${STAGES:-"test smoke bench launches full"}
for s in $STAGES; do
  case $s in
    test)  timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q --maxfail=40 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?";;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?";;
    bench) timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ncu_launch_bench.log 2>&1; echo "launches rc=$?";;
    full) timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-gemm} -s ${NCU_S:-19} -c ${NCU_C:-3} -o gpurun_out/prof_full -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
           # summaries here (the full report can exceed what gpurun copies back)
           python tools/ncu_summary.py gpurun_out/launches.csv gpurun_out/prof_full.ncu-rep > gpurun_out/ncu_summary.txt 2>&1
           bash tools/ncu_brief.sh gpurun_out/prof_full.ncu-rep > gpurun_out/ncu_brief.txt 2>&1
           python tools/ncu_stalls.py gpurun_out/prof_full.ncu-rep 40 > gpurun_out/ncu_stalls.txt 2>&1
           [ -n "$KEEP_REP" ] || rm -f gpurun_out/prof_full.ncu-rep;;
  esac
done
