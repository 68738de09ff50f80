for c in vgg_b64 alexnet_b128; do
  for mb in 1,4 4,6 1,4 4,6; do
    TPX_MOVE_MINB=$mb timeout 300 python bench.py --config $c --no-cpu-baseline --no-variants 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', '$mb', round(d['value']), round(d['ms_per_step'],3), d['clocks']['reasons'])"
  done
done
