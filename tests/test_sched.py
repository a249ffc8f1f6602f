"""Iteration stream: the C++ batch former + KV page allocator (duet_sched_*), host only.

Invariants checked on seeded random traces (P:184 decode-first chunked prefill, P:302, P:335 look-ahead
slots, S:376 KV-capacity admission): token budget, decode-first, pages never shared and always
conserved, page tables covering c + k_max for decodes and c + q for prefill chunks, FIFO admission,
every request finishing with exactly prompt + output tokens, and determinism."""
import numpy as np
import pytest

import paper_2511_04791_b200 as D


def _trace(seed, n=40, max_prompt=3000, max_out=60):
    rng = np.random.default_rng(seed)
    t = np.cumsum(rng.gamma(0.25, 4.0, size=n) * 1e-3)     # bursty (CV = 2) arrivals
    return [(i, int(rng.integers(1, max_prompt)), int(rng.integers(1, max_out)), float(t[i])) for i in range(n)]


def _run(trace, k_choices=(1, 2, 3), seed=0, **cfg):
    rng = np.random.default_rng(seed)
    s = D.Sched(**cfg)
    P, k_max, budget, max_batch = cfg["page_size"], cfg["k_max"], cfg["token_budget"], cfg["max_batch"]
    for r in trace:
        s.add(*r)
    now, log = 0.0, []
    total_tokens = 0
    admitted_order = []
    meta = {r[0]: (r[1], r[2]) for r in trace}     # id -> (prompt, output)
    running = {}                                   # id -> tokens generated, for requests past their prompt
    for _ in range(100000):
        it = s.next(now)
        if not it["prefill"] and not it["decode"]:
            if it["unfinished"] == 0:
                break
            assert it["next_arrival"] >= 0
            now = max(now, it["next_arrival"])
            continue
        n_dec, n_pre = len(it["decode"]), len(it["prefill"])
        tokens = sum(q for _, q, _ in it["prefill"]) + n_dec
        assert tokens <= budget and n_dec <= max_batch
        tab = it["table"]
        # pages: distinct across and within live rows, page tables cover the slots the step touches
        used = []
        for i, (rid, q, c) in enumerate(it["prefill"]):
            need = -(-(c + q) // P)
            assert all(p >= 0 for p in tab[i][:need])
            used.extend(tab[i][:need])
            if c == 0:
                admitted_order.append(rid)
        for j, (rid, c) in enumerate(it["decode"]):
            need = -(-(c + k_max) // P)
            used.extend(tab[n_pre + j][:need])
        assert len(used) == len(set(used))
        # decode-first: every request past its prompt and not finished has a decode row, so
        # no running decode is ever skipped (and none waits while holding its pages)
        assert sorted(rid for rid, _ in it["decode"]) == sorted(running)
        assert len(running) + n_pre <= max_batch
        for rid, c in it["decode"]:                 # the decode input is the last generated token
            assert c == meta[rid][0] + running[rid] - 1
        k = int(rng.choice(k_choices))
        toks, fin = s.commit(k)
        for rid in list(running):
            running[rid] += min(k, meta[rid][1] - running[rid])
            if running[rid] >= meta[rid][1]:
                del running[rid]
        for rid, q, c in it["prefill"]:
            if c + q == meta[rid][0] and meta[rid][1] > 1:
                running[rid] = 1                    # the prompt's last position yields token 1
        total_tokens += toks
        log.append((tuple(it["prefill"]), tuple(it["decode"]), toks))
        now += 1e-3
    assert s.free_pages() == cfg["n_pages"]             # every page returned
    s.close()
    return log, total_tokens, admitted_order


CFG = dict(page_size=16, n_pages=2048, token_budget=1024, max_batch=32, max_prefill_seqs=8, k_max=4,
           max_pages_per_seq=256)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_sched_invariants_and_token_accounting(seed):
    trace = _trace(seed)
    log, total, order = _run(trace, seed=seed, **CFG)
    assert total == sum(p + o for _, p, o, _ in trace)   # every prompt token prefilled, every output produced
    assert order == sorted(order)                        # FIFO admission (ids follow arrival order)


@pytest.mark.parametrize("max_batch", [2, 5])
def test_sched_decodes_never_exceed_max_batch(max_batch):
    """More arrivals than max_batch: admission waits, so every running decode gets a row each iteration."""
    trace = _trace(11, n=30, max_prompt=400, max_out=40)
    log, total, order = _run(trace, seed=3, **dict(CFG, max_batch=max_batch))
    assert total == sum(p + o for _, p, o, _ in trace)
    assert max(len(d) for _, d, _ in log) <= max_batch


def test_sched_deterministic():
    trace = _trace(5)
    a = _run(trace, seed=9, **CFG)
    b = _run(trace, seed=9, **CFG)
    assert a == b


def test_sched_capacity_admission_no_overcommit():
    """A pool that fits only one long request at a time: the second waits until the first finishes."""
    cfg = dict(CFG, n_pages=200)
    s = D.Sched(**cfg)
    s.add(0, 3000, 10, 0.0)   # needs ceil(3014 / 16) = 189 pages
    s.add(1, 200, 5, 0.0)     # needs 14 pages: does not fit next to request 0 (189 + 14 > 200)
    it = s.next(0.0)
    assert [e[0] for e in it["prefill"]] == [0]
    seen_second_early = False
    for _ in range(100):
        s.commit(1)
        it = s.next(0.0)
        if not it["prefill"] and not it["decode"]:
            break
        ids_pre = [e[0] for e in it["prefill"]]
        ids_dec = [e[0] for e in it["decode"]]
        if 1 in ids_pre and 0 in ids_dec:
            seen_second_early = True
    assert not seen_second_early
    assert s.free_pages() == 200


def test_sched_errors():
    s = D.Sched(**CFG)
    with pytest.raises(D.DuetError):
        s.add(0, 10_000, 10, 0.0)      # 10014 tokens > 256 pages x 16
    s.add(1, 10, 2, 1.0)
    with pytest.raises(D.DuetError):
        s.add(2, 10, 2, 0.5)           # arrivals must be non-decreasing
    with pytest.raises(D.DuetError):
        s.commit(1)                    # no open iteration
