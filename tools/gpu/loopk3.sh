for st in cfg2_mlp5x8192_b512.loop.k3 cfg2_mlp5x8192_b512.loop.k2 cfg2_mlp5x8192_b512.loop.k1 cfg2_mlp5x8192_b512.opt.k0; do
  timeout 300 python tools/step_profile.py $st 6 2>&1 | head -9
done
python tools/desc_probe.py 2>&1 | head -3
