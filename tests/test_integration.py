"""INTEGRATION.md's reference-side adapter, compiled for real (integration/*.cpp, built by
oracle/Makefile against the UNMODIFIED reference sources and linked with libtpx.so): the
reference's own API end to end -- gen_mlp -> kcuts / preset_assignment -> place_k ->
build_execution_graph -- into the B200 executor through the C ABI.

CPU: the B200 lowering's per-phase fetch bytes, summed over every rank of a 2^k-rank job (NCCL
and peer modes), equal the reference's simulate_traffic phase totals (proj/src/simulator.cpp:
11-49), and the flat-hierarchy time model est_seconds = sum over phases of bytes / bandwidth
equals the reference's.
GPU: execute_numeric_b200 (fp32-accurate) against the reference's serial_execute with the
reference's own metric (simulator.cpp:129-147), gate 2e-2 (chained)."""
import json
import os
import subprocess

import pytest

from oracle import ref

CASES = [("64", "1", "opt", ["1024"] * 4), ("64", "2", "data", ["1024"] * 4), ("64", "3", "opt", ["256"] * 4),
         ("32", "2", "hybrid", ["128"] * 5), ("16", "2", "model", ["64"] * 3)]


def adapter():
    if not os.path.exists(ref.ADAPTER):
        if not os.path.isdir("/root/reference/proj/src"):
            pytest.skip("adapter not built and the reference sources are absent")
        ref.build()
    return ref.ADAPTER


def run(args):
    out = subprocess.run([adapter()] + args, capture_output=True, text=True, timeout=600)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    return out.returncode, d


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"b{c[0]}.k{c[1]}.{c[2]}")
def test_adapter_phase_bytes_match_simulate_traffic(case):
    b, k, mode, dims = case
    rc, d = run([b, k, mode] + dims)
    assert rc == 0 and d["pass"], d
    assert d["phase_bytes_match"] and d["phase_bytes_match_peer"]


def test_flat_time_model_matches_reference():
    """est_seconds for a flat NVSwitch level (the per-phase bytes over the level bandwidth,
    simulator.cpp:40-47) recomputed from the executor's per-phase bytes."""
    if not ref.available():
        pytest.skip("reference library not built")
    from paper_1805_04170_b200.executor import Context, PlanExecutor
    g = ref.gen_mlp(64, [256] * 4)
    for mode, k in (("opt", 2), ("data", 3)):
        text = ref.plan(g, mode, k)
        t = ref.simulate_traffic(text)
        bw = json.loads(ref.flat_hierarchy(k))["levels"][0]["bandwidth_bytes_per_s"]
        ours = 0.0
        phases = {}
        for r in range(1 << k):
            for ph, v in PlanExecutor(Context.host_only(r, 1 << k), text).describe()["per_phase_fetch_bytes_in"].items():
                phases[ph] = phases.get(ph, 0) + v
        ours = sum(v / bw for v in phases.values())
        assert ours == pytest.approx(t["est_seconds"], rel=1e-12)


@pytest.mark.gpu
def test_adapter_execute_numeric_b200_on_gpu():
    rc, d = run(["64", "1", "opt"] + ["1024"] * 4 + ["--gpu"])
    assert rc == 0, d
    assert d["numeric"]["values"] > 0
    assert d["numeric"]["max_rel"] <= 2e-2, d
