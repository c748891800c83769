"""NEXT(4) host control plane (include/grpo_transfer_queue.h), -m "not gpu":
SPEC transfer_queue worked examples and audits on the C++
sliding window + TransferQueue, and a small streaming-rollout simulation whose
batches satisfy C2/C3 as checked by the oracle's validate."""
import numpy as np
import pytest

import oracle.oracle as O
from paper_2604_26256_b200 import GrpoError
from paper_2604_26256_b200.transfer_queue import TransferQueue


def test_push_under_current_version_accepted():
    q = TransferQueue(G=4, K=3, first_version=1)
    q.dispatch(1, 1)
    q.push(0, 0, 1, 10, 1.0)                      # S:320 [TRIVIAL]
    assert q.stats()["queued"] == 1


def test_push_for_evicted_version_is_fatal():
    q = TransferQueue(G=1, K=1, first_version=1)   # version evicted from W
    adv, _, _ = q.advance(2)
    assert adv
    with pytest.raises(GrpoError) as e:
        q.push(0, 0, 1, 5, 0.0)
    assert e.value.status == 1                     # GRPO_ERR_VALIDATION


def test_fifo_across_interleaved_versions():
    """pushes from two versions interleaved keep arrival order."""
    q = TransferQueue(G=2, K=2, first_version=1)
    q.dispatch(1, 2)
    q.advance(2)
    q.dispatch(2, 2)
    q.push(10, 7, 2, 3, 1.0)
    q.push(11, 9, 1, 4, 0.0)
    q.push(12, 7, 1, 5, 0.0)
    q.push(13, 9, 2, 6, 1.0)
    b = q.form_batch(4, v_theta=2)
    assert b.request_ids.tolist() == [10, 12, 11, 13]   # prompt 7 arrived first
    assert b.group_ids.tolist() == [0, 0, 1, 1]
    assert b.version_ids.tolist() == [2, 1, 1, 2]       # a group may span versions (P:7)


def test_batch_of_two_oldest_groups():
    """3 complete groups of G=4, tbs=8 -> the 2 oldest groups, 1 group remains."""
    q = TransferQueue(G=4, K=2, first_version=1)
    q.dispatch(1, 12)
    rid = 0
    for p in (5, 3, 8):
        for _ in range(4):
            q.push(rid, p, 1, 7, 0.5)
            rid += 1
    b = q.form_batch(8, v_theta=1)
    assert b is not None and set(b.prompt_ids.tolist()) == {5, 3}
    st = q.stats()
    assert st["queued"] == 4 and st["consumed"] == 8 and st["pushed"] == 12


def test_incomplete_group_forms_nothing():
    """7 of a group's 8 members queued, tbs=8 -> none."""
    q = TransferQueue(G=8, K=1, first_version=0)
    q.dispatch(0, 7)
    for i in range(7):
        q.push(i, 0, 0, 3, 1.0)
    assert q.form_batch(8, v_theta=0) is None
    assert q.stats()["queued"] == 7


def test_bad_tbs_is_a_precondition_violation():
    """tbs=0 (and tbs not a multiple of G) -> precondition violation."""
    q = TransferQueue(G=4, K=1, first_version=0)
    for tbs in (0, 6):
        with pytest.raises(GrpoError) as e:
            q.form_batch(tbs, v_theta=0)
        assert e.value.status == 2


def test_window_protocol_examples():
    """W={3,2,1}, K=3: drained oldest -> {4,3,2}; 2 in flight -> blocked(2);
    W={2,1}, K=3 -> advance(3) unconditionally; non-consecutive versions are fatal."""
    q = TransferQueue(G=1, K=3, first_version=1)
    assert q.advance(2)[0] and q.stats()["window"] == [2, 1]
    assert q.advance(3)[0] and q.stats()["window"] == [3, 2, 1]
    q.dispatch(1, 2)
    assert q.advance(4) == (False, 2, 0)
    q.push(0, 0, 1, 5, 0.0)
    q.push(1, 1, 1, 5, 0.0)
    assert q.advance(4) == (False, 0, 2)            # collected but not yet forwarded
    assert q.form_batch(2, v_theta=3) is not None
    assert q.advance(4)[0] and q.stats()["window"] == [4, 3, 2]
    with pytest.raises(GrpoError):
        q.advance(6)


def test_c3_checked_at_formation():
    q = TransferQueue(G=1, K=1, first_version=5)
    q.dispatch(5, 1)
    q.push(0, 0, 5, 4, 1.0)
    with pytest.raises(GrpoError) as e:
        q.form_batch(1, v_theta=7)                   # staleness 2 > K = 1
    assert e.value.status == 1
    assert q.form_batch(1, v_theta=6) is not None    # staleness 1 = K passes (Z8)


@pytest.mark.parametrize("seed", range(5))
@pytest.mark.parametrize("K", [1, 2, 3])
def test_streaming_rollout_simulation(seed, K):
    """A small multi-version streaming rollout: RBS > TBS prompts are dispatched
    under the newest version, long-tailed responses complete over several steps, the trainer
    consumes TBS trajectories per step and the window advances after each step.  Audits:
    every batch has exactly TBS trajectories in complete groups (C2), staleness <= K (C3),
    nothing is dropped (pushed == consumed + queued), and the oracle's validate passes."""
    rng = np.random.default_rng(seed)
    G, TBS, RBS = 4, 16, 6
    q = TransferQueue(G=G, K=K, first_version=0)
    v_theta, rid, pid = 0, 0, 0
    running = []   # (finish_step, request_id, prompt_id, version, length, reward)
    step = 0
    batches = 0
    while batches < 12 and step < 200:
        # the rollout keeps RBS prompts' worth of requests in flight under the newest version
        while len(running) < RBS * G:
            q_p = rng.random()
            for _ in range(G):
                L = int(min(1 + rng.lognormal(3.0, 1.0), 400))
                running.append((step + 1 + L // 60, rid, pid, v_theta, L, float(rng.random() < q_p)))
                rid += 1
            q.dispatch(v_theta, G)
            pid += 1
        done = [r for r in running if r[0] <= step]
        running = [r for r in running if r[0] > step]
        for _, r_id, p_id, ver, L, R in done:
            q.push(r_id, p_id, ver, L, R)
        b = q.form_batch(TBS, v_theta=v_theta)
        if b is not None:
            batches += 1
            assert len(b.lengths) == TBS
            assert np.all(np.bincount(b.group_ids) == G)
            cu = b.cu_seqlens
            val = O.validate(b.version_ids, cu, b.group_ids, np.zeros(cu[-1], np.int64),
                             P=TBS // G, V=2, G=G, tbs=TBS, v_theta=v_theta, K=K)
            assert val["summary"]["valid"] == 1, val["summary"]
            # training step done: try to move to the next version (may block on stragglers)
            adv, _, _ = q.advance(v_theta + 1)
            if adv:
                v_theta += 1
        step += 1
        st = q.stats()
        assert st["pushed"] == st["consumed"] + st["queued"]
        assert st["max_staleness"] <= K and st["window_size"] <= K
    assert batches == 12
