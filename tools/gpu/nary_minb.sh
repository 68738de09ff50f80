for st in cfg2_mlp5x8192_b512.loop.k3 cfg2_mlp5x8192_b512.data.k3 alexfc_b128.opt.k3; do
  for mb in 2,3 3,3 4,3 2,4 2,6 2,3; do
    echo "== $st TPX_NARY_MINB=$mb"; TPX_NARY_MINB=$mb timeout 300 python tools/step_profile.py $st 0 2>&1 | head -4 | grep -E "steps|nary"
  done
done
