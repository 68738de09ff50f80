mkdir -p gpurun_out
export SHAPES="fwd,bwd_x"
timeout 600 python tools/epi_sweep.py base whole=23:1 st5=4:5 st4=4:4 rr0=20:0 nodyn=10:0 > gpurun_out/sweep_fwd.txt 2>&1; echo "sweep $?"
timeout 300 python tools/gemm_trace.py 512,8192,8192,0,0 512,8192,8192,0,1 8192,8192,512,1,0 > gpurun_out/trace_fwd.txt 2>&1; echo "trace $?"
cat gpurun_out/sweep_fwd.txt gpurun_out/trace_fwd.txt
