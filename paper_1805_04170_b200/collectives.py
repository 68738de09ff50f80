"""Which collective each phase of a plan is (host-side analysis of the plan document).

The reference moves data only through `fetch` nodes (proj/src/simulator.cpp:88-93) whose pieces
come from Builder::assemble (proj/src/execgraph.cpp:101-188); a phase (`<op>:in<j>` /
`<op>:out`, execgraph.cpp:41-47) converts one tensor between two tilings.  Seen per phase, the
message set of a conversion is one of the classic collectives over groups of devices that differ
only in some cut bits (device id = cut bits, outermost cut = MSB, proj/src/tiling.cpp:200-210):

    all_gather      every device receives every group peer's whole block      (P -> r)
    all_to_all      every device receives a different part of each peer       (P_i -> P_j)
    reduce_scatter  partials summed into disjoint blocks (reduce_partial)     (red -> P)
    all_reduce      every device sums all partials over the same block        (red -> r)
    gather / mixed  anything else (e.g. uneven or partial groups)

The executor does not need the label (peer mode pulls every piece in one launch per phase, the
NCCL fallback pairs send/recv per piece); `describe_collectives` reports it next to the bytes so a
plan can be read as "AllGather over groups of 8 on bits 0b111" (bench.py, tests/test_collectives.py).
"""
from __future__ import annotations

from collections import defaultdict
from typing import Dict, List


def _vol(region) -> int:
    v = 1
    for lo, hi in region:
        v *= hi - lo
    return v


def _disjoint(a, b) -> bool:
    return any(ahi <= blo or bhi <= alo for (alo, ahi), (blo, bhi) in zip(a, b))


def classify_phases(plan: dict) -> List[Dict]:
    nodes = {n["id"]: n for n in plan["nodes"]}
    by_phase: Dict[str, List[dict]] = defaultdict(list)
    order: List[str] = []
    for n in plan["nodes"]:
        if n["phase"] not in by_phase:
            order.append(n["phase"])
        by_phase[n["phase"]].append(n)
    out = []
    for ph in order:
        fetches = [n for n in by_phase[ph] if n["kind"] == "fetch"]
        if not fetches:
            continue
        reduces = [n for n in by_phase[ph] if n["kind"] == "reduce_partial"]
        # groups: connected components of the (receiver, sender) graph
        parent = {}

        def find(x):
            parent.setdefault(x, x)
            while parent[x] != x:
                parent[x] = parent[parent[x]]
                x = parent[x]
            return x

        for f in fetches:
            parent[find(f["device"])] = find(f["src_device"])
        comps = defaultdict(set)
        for d in list(parent):
            comps[find(d)].add(d)
        groups = sorted(sorted(c) for c in comps.values())
        sizes = sorted({len(g) for g in groups})
        bits = 0
        for g in groups:
            for d in g:
                bits |= d ^ g[0]
        recv = defaultdict(lambda: defaultdict(list))  # dst -> src -> pieces
        for f in fetches:
            recv[f["device"]][f["src_device"]].append(f)
        whole = all(f["region"] == nodes[f["sources"][0]]["region"] for f in fetches)
        full_mesh = all(len(recv[d]) == len(g) - 1 for g in groups for d in g)
        if reduces:
            regs = defaultdict(list)
            for r in reduces:
                regs[r["device"]].append(r["region"])
            same = all(len({str(regs[d]) for d in g if d in regs}) == 1 for g in groups)
            disj = all(_disjoint(regs[a][0], regs[b][0]) for g in groups for i, a in enumerate(g) for b in g[i + 1:]
                       if a in regs and b in regs)
            pattern = "all_reduce" if same else "reduce_scatter" if disj else "reduce_mixed"
        elif whole and full_mesh:
            pattern = "all_gather"
        elif full_mesh:
            pattern = "all_to_all"
        else:
            pattern = "gather" if whole else "mixed"
        out.append({"phase": ph, "pattern": pattern, "group_sizes": sizes, "groups": len(groups),
                    "cut_bits": bits, "pieces": len(fetches), "bytes": sum(f["bytes"] for f in fetches)})
    return out


def describe_collectives(plan: dict) -> Dict[str, Dict]:
    """pattern -> {phases, bytes} totals of a plan (bench.py reports it per plan)."""
    tot: Dict[str, Dict] = {}
    for p in classify_phases(plan):
        t = tot.setdefault(p["pattern"], {"phases": 0, "bytes": 0})
        t["phases"] += 1
        t["bytes"] += p["bytes"]
    return tot
