for st in cfg2_mlp5x8192_b512.data.k3 cfg2_mlp5x8192_b512.loop.k3; do
  timeout 300 python tools/step_profile.py $st 12 2>&1 | head -20
done
