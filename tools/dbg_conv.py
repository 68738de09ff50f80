import gzip, sys
sys.path.insert(0, '.')
from paper_1805_04170_b200.executor import Context, PlanExecutor
text = gzip.open('tests/golden/alexr_conv_b4.data.k1.s7.plan.json.gz', 'rt').read()
ex = PlanExecutor(Context(0), text, precision=int(sys.argv[1]) if len(sys.argv) > 1 else 0, flags=1)
import json
d = ex.describe()
for s in d['main']['steps']:
    if s['kind'] == 'gemm': print(s)
ex.init_inputs(7)
ex.execute()
ex.synchronize()
print("ok")
