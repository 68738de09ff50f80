"""Host-side tile scheduler of the persistent tcgen05 GEMM (csrc/gemm.cu gemm_schedule).

CPU only: the schedule is built on the host and exported through the C ABI
(tpx_gemm_schedule).  Properties checked for every shape the BASELINE configs lower to, plus
edge shapes:
  * every output tile's k-blocks are covered exactly once, by one head/whole segment and its
    partial segments in k order with consecutive slots (deterministic reduction order);
  * slots are unique;
  * deadlock freedom: a CTA never holds a waiting (head) segment before a partial-producing
    one, so every wait targets work that does not itself wait;
  * the k-blocks are balanced over at most num_sms CTAs.
"""
import itertools
import random

import pytest

from paper_1805_04170_b200 import native

WHOLE, HEAD, PART = 0, 1, 2


def _check(nprob, P, Q, K, bn, sms=148, force=0, max_kb=0):
    S = native.gemm_schedule(nprob, P, Q, K, bn, sms, force, max_kb)
    tiles_p, tiles_q, kbt = -(-P // 128), -(-Q // bn), -(-K // 32)
    assert 1 <= S["grid"] <= max(sms, force)
    segs, off = S["segs"], S["seg_off"]
    assert off[0] == 0 and off[-1] == len(segs)
    by_tile = {}
    for cta in range(S["grid"]):
        kinds = []
        for i in range(off[cta], off[cta + 1]):
            prob, tp, tq, kb0, kb1, kind, slot, nparts = segs[i]
            assert 0 <= prob < nprob and 0 <= tp < tiles_p and 0 <= tq < tiles_q
            assert 0 <= kb0 <= kb1 <= kbt
            if max_kb:
                assert kb1 - kb0 <= max_kb
            by_tile.setdefault((prob, tp, tq), []).append((kb0, kb1, kind, slot, nparts))
            kinds.append(kind)
        # no HEAD before a PART inside one CTA's list
        if PART in kinds and HEAD in kinds:
            assert max(i for i, k in enumerate(kinds) if k == PART) < min(i for i, k in enumerate(kinds) if k == HEAD)
    assert len(by_tile) == nprob * tiles_p * tiles_q
    slots = []
    for t, ss in by_tile.items():
        ss.sort()
        assert ss[0][0] == 0 and ss[-1][1] == kbt, t
        for a, b in zip(ss, ss[1:]):
            assert a[1] == b[0], t
        if len(ss) == 1:
            assert ss[0][2] == WHOLE
        else:
            head = ss[0]
            assert head[2] == HEAD and head[4] == len(ss) - 1
            for j, s in enumerate(ss[1:]):
                assert s[2] == PART and s[3] == head[3] + j
                slots.append(s[3])
    assert sorted(slots) == list(range(S["nslots"]))
    work = [sum(segs[i][4] - segs[i][3] for i in range(off[c], off[c + 1])) for c in range(S["grid"])]
    return S, work


BASELINE_SHAPES = [
    # (nprob, P, Q, K, bn)  in kernel orientation (P = 128-row tiles)
    (1, 512, 8192, 8192, 256),     # cfg2 k=0 fwd / bwd_x
    (1, 8192, 8192, 512, 256),     # cfg2 k=0 bwd_w
    (1, 8192, 64, 8192, 64),       # cfg2 n=8 fwd (swapped, M=64)
    (8, 8192, 64, 8192, 64),       # cfg2 k=3 on one GPU: 8 logical devices batched
    (1, 1024, 8192, 512, 256),     # cfg2 n=8 bwd_w
    (1, 32768, 32, 32768, 32),     # cfg5 (M=4 per GPU at n=8 pads to 32)
    (1, 1024, 64, 1024, 64),       # cfg1
    (2, 1024, 32, 1024, 32),       # cfg1 k=1
    (1, 4096, 128, 9216, 128),     # AlexNet FC6 b128
    (1, 1000, 128, 4096, 128),     # AlexNet FC8 (N=1000 edge)
]


@pytest.mark.parametrize("shape", BASELINE_SHAPES)
def test_schedule_baseline_shapes(shape):
    S, work = _check(*shape)
    avg = sum(work) / len(work)
    assert max(work) <= avg * 1.12 + 16, (max(work), avg)


def test_small_m_groups_share_the_streamed_operand():
    # 32 columns of 4 P-tiles on 37 groups: >= 80 % of the groups get a whole column
    S, _ = _check(1, 512, 8192, 8192, 256)
    assert S["group"] == 4 and not S["stream_k"] and S["grid"] == 128
    # 16 columns on 37 groups: stream-K, every CTA busy
    S, _ = _check(1, 512, 4096, 8192, 256)
    assert S["group"] == 4 and S["stream_k"] and S["grid"] == 148


def test_many_tiles_use_whole_tiles():
    S, work = _check(1, 8192, 8192, 512, 256)
    assert not S["stream_k"] and S["nslots"] == 0
    assert max(work) - min(work) <= 16


@pytest.mark.parametrize("P,Q,K,bn", [(128, 128, 32, 128), (1, 1, 0, 32), (200, 300, 100, 256),
                                      (1000, 136, 72, 256), (128, 32, 32 * 1000, 32), (64, 64, 8, 64)])
def test_schedule_edges(P, Q, K, bn):
    _check(1, P, Q, K, bn)


def test_schedule_random_and_forced():
    rng = random.Random(5)
    for _ in range(60):
        nprob = rng.choice([1, 2, 4, 8])
        P, Q = rng.randint(1, 3000), rng.randint(1, 3000)
        K = rng.randint(0, 20000)
        bn = rng.choice([32, 64, 128, 256])
        sms = rng.choice([1, 3, 16, 148])
        _check(nprob, P, Q, K, bn, sms)
    for force in [1, 2, 7, 37]:
        _check(1, 512, 8192, 8192, 256, 148, force)


def test_long_k_few_tiles_caps_the_cut():
    """A 64 x 27 conv grad_weight over 61696 columns (one tile, 1928 k-blocks): the tile is cut
    into ~sqrt(kb * k-block bytes / tile bytes) ~ 49 parts, not one per SM, so the head's serial
    sum of partials stays as short as each part's operand reads."""
    S, work = _check(1, 64, 27, 61696, 32)
    assert S["stream_k"] and 30 <= S["grid"] <= 64, S["grid"]
    assert S["nslots"] == S["grid"] - 1


@pytest.mark.parametrize("shape", BASELINE_SHAPES + [(1, 256, 3456, 100352, 256), (1, 128, 27, 61696, 32)])
@pytest.mark.parametrize("max_kb", [8, 16])
def test_bounded_chains(shape, max_kb):
    """3xTF32 schedules: every segment accumulates at most max_kb k-blocks in TMEM (the tensor
    cores' fp32 accumulation error grows with the chain length); coverage, slot order and the
    no-head-before-partial rule still hold, and the k-work stays balanced."""
    S, work = _check(*shape, max_kb=max_kb)
    kbt = -(-shape[3] // 32)
    if kbt > max_kb:
        assert S["stream_k"] and S["nslots"] > 0
    avg = sum(work) / len(work)
    assert max(work) <= avg + 2 * max_kb, (max(work), avg)
