set -x; mkdir -p gpurun_out
SHAPES="bwd_w" timeout 900 python tools/epi_sweep.py base "o2=15:2" "o1=15:1" "o3=15:3" "o2s5=15:2,16:5" "o3s4=15:3,4:4" > gpurun_out/r2_epi_sweep3.txt 2>&1; grep sweep gpurun_out/r2_epi_sweep3.txt
