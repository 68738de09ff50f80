set -x; mkdir -p gpurun_out/tmp
for cfg in "fwd128:128 8192 8192 0 0 1" "bww1024:1024 8192 512 1 0 3,6"; do
  name=${cfg%%:*}; shape=${cfg#*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm -s 3 -c 1 -f -o gpurun_out/tmp/r2_ncu_$name python tools/gemm_check.py --one $shape > gpurun_out/r2_ncu_$name.log 2>&1
  ncu -i gpurun_out/tmp/r2_ncu_$name.ncu-rep --page raw --csv > gpurun_out/r2_ncu_${name}_raw.csv 2>&1
  python tools/ncu_stalls.py gpurun_out/tmp/r2_ncu_$name.ncu-rep 40 > gpurun_out/r2_ncu_${name}_stalls.txt 2>&1
  TPX_GEMM_KNOBS= python -c "
import sys; sys.path.insert(0,'.')
from tools.gemm_check import run
from paper_1805_04170_b200 import native
import torch
" 
done
python - <<'PY'
import sys; sys.path.insert(0,'.')
import torch
from paper_1805_04170_b200 import native
for shp, epi in (((128,8192,8192,False,False),[1]), ((1024,8192,512,True,False),[3,6]), ((64,8192,8192,False,False),[1])):
    M,N,K,ta,tb=shp
    A=torch.rand((K,M) if ta else (M,K),device='cuda'); B=torch.rand((N,K) if tb else (K,N),device='cuda')
    C=torch.empty(M,N,device='cuda'); W=torch.rand(M,N,device='cuda'); outs=[torch.empty(M,N,device='cuda') for _ in epi]
    native.gemm(A,B,ta,tb,C,epi=[(op,0.01,W if op>=4 else None,o) for op,o in zip(epi,outs)]); torch.cuda.synchronize()
    print(shp, native.last_launch())
PY
rm -rf gpurun_out/tmp
