"""Multi-process (world_size 2, gloo, CPU) check of the N>1 path's host logic: each process
lowers the plan for its own rank (logical device d -> rank (d * world) >> k), the ranks
exchange their lowered programs over torch.distributed, and every NCCL exchange group must
pair up across ranks with the planner's fetch bytes (what a real 2-GPU run relies on)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.conftest import golden_stems, load_golden, stem_id

CASES = [s for s in golden_stems() if stem_id(s).split(".")[0] in
         ("cfg1_mlp3x1024_b64", "cfg2r_mlp5x256_b64", "fcr_alexnet_b32", "cnnr_train_b16",
          "mlp_train_d3", "cnn_train") and ".k0." not in s]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, stems, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1805_04170_b200.executor import Context, PlanExecutor
        from tests.test_abi import check_pairing
        out = []
        for stem in stems:
            text, P, _, _ = load_golden(stem)
            ex = PlanExecutor(Context.host_only(rank, world), text)
            mine = {"desc": ex.describe(), "stats": ex.stats()}
            gathered = [None] * world
            dist.all_gather_object(gathered, mine)
            if rank == 0:
                check_pairing([g["desc"] for g in gathered])
                tot = sum(g["stats"]["rank_fetch_bytes_in"] for g in gathered)
                assert tot == P["fetch_bytes_total"], stem
                xin = sum(g["stats"]["rank_xrank_bytes_in"] for g in gathered)
                xout = sum(g["stats"]["rank_xrank_bytes_out"] for g in gathered)
                assert xin == xout
                out.append((stem_id(stem), tot, xin))
        dist.barrier()
        if rank == 0:
            q.put(("ok", out))
    except Exception as e:  # noqa: BLE001
        q.put(("err", f"rank {rank}: {e!r}"))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_programs_pair_over_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, CASES, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    status, payload = q.get(timeout=10)
    assert status == "ok", payload
    assert len(payload) == len(CASES)
    # some plans really cross the rank boundary
    assert any(x > 0 for _, _, x in payload)
    for p in procs:
        assert p.exitcode == 0
