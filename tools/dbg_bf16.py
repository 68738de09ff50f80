import sys, json
sys.path.insert(0, '.')
from tests.conftest import golden_stems, load_golden
from oracle import tileplan_oracle as O
from paper_1805_04170_b200.executor import Context, PlanExecutor
stem = [s for s in golden_stems() if "mlp_train_d2_bf16.data.k2" in s][0]
text, P, vals, seed = load_golden(stem)
serial = O.serial_execute(P["graph"], seed)
v = O.execute_nodes(P, serial)
ctx = Context(0)
ex = PlanExecutor(ctx, text, precision=0, flags=0)
d = ex.describe()
ex.init_inputs(seed)
ex.synchronize()
for op in P["graph"]["ops"]:
    for t in op["inputs"]:
        for h in P["holders"][t]:
            ex.write_node(h, v[h])
    steps = [s for s in d["main"]["steps"] if s["op"] == op["id"]]
    print("op", op["id"], json.dumps(steps)[:600], flush=True)
    ex.execute_op(op["id"])
    ex.synchronize()
    print("  ok", flush=True)
