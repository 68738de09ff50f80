python tools/launch_info.py 128,8192,8192,0,0,1 64,8192,8192,0,0,1 256,8192,8192,0,0,1 512,8192,8192,0,0,1 1024,8192,512,1,0,3:6 2048,8192,512,1,0,3:6 64,8192,8192,0,1,2
for st in 3 5 6 8; do TPX_GEMM_KNOBS=4:$st python tools/gemm_check.py --one 128 8192 8192 0 0 1 | tail -1; done
