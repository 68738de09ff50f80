for st in alexconv_b128.opt.k0 vggconv_b64.opt.k0; do
  for mb in 4,4 4,5 4,6 4,4; do
    echo "== $st TPX_MOVE_MINB=$mb"; TPX_MOVE_MINB=$mb timeout 300 python tools/step_profile.py $st 0 2>&1 | head -5 | grep -E "steps|col2im"
  done
done
