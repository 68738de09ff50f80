for kn in "" "9:128" "6:1"; do
  for shp in "512 8192 8192 0 0 1" "512 8192 8192 0 1 2" "8192 8192 512 0 1 -" "8192 8192 512 1 0 -"; do
    TPX_GEMM_KNOBS=$kn python tools/gemm_check.py --one $shp | tail -1 | sed "s/^/knob=$kn /"
  done
done
python - <<'PY'
import sys; sys.path.insert(0,'.')
from tools.gemm_check import bench
for shp in ((512,8192,8192,False,False),(512,8192,8192,False,True),(8192,8192,512,False,True),(8192,8192,512,True,False)):
    r=sorted(bench(*shp, precision=2, epi=None) for _ in range(5))[2]
    print("bf16", shp, f"{r[0]*1e3:.1f} us {r[1]:.0f} TF/s")
PY
