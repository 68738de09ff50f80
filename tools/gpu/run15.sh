set -x; mkdir -p gpurun_out
SHAPES="bwd_w" timeout 900 python tools/epi_sweep.py base "ts1=18:1" "ts2=18:2" "ts1o2=18:1,15:2" "ts1nl=18:1,12:0" > gpurun_out/r2_epi_sweep4.txt 2>&1; grep sweep gpurun_out/r2_epi_sweep4.txt; tail -3 gpurun_out/r2_epi_sweep4.txt
for kn in "18:1" "18:2"; do TPX_GEMM_KNOBS=$kn timeout 300 python tools/gemm_check.py --one 8192 8192 512 1 0 3,6 2>&1 | tail -1; done
